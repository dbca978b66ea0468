// Host-DRAM probe: in-place AdamW-like pass over separate p / m / v arrays (+ bf16 g) vs an
// interleaved [p m v] record layout (+ bf16 g), same bytes per parameter (28), OpenMP dynamic
// 64 KiB chunks. g++ -O3 -march=native -fopenmp host_layout_probe.cpp -o probe; ./probe [Mparams] [threads]
#include <omp.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

int main(int argc, char** argv) {
    const size_t n = (argc > 1 ? atol(argv[1]) : 400) * 1000000ul;
    const int th = argc > 2 ? atoi(argv[2]) : omp_get_num_procs();
    float *p = (float*)aligned_alloc(4096, n * 4), *m = (float*)aligned_alloc(4096, n * 4), *v = (float*)aligned_alloc(4096, n * 4);
    float* pmv = (float*)aligned_alloc(4096, n * 12);
    uint16_t* g = (uint16_t*)aligned_alloc(4096, n * 2);
#pragma omp parallel for num_threads(th)
    for (size_t i = 0; i < n; ++i) { p[i] = 0.01f; m[i] = 0; v[i] = 0; pmv[3 * i] = 0.01f; pmv[3 * i + 1] = 0; pmv[3 * i + 2] = 0; g[i] = 0x3c00; }
    const float b1 = 0.9f, b2 = 0.999f, lr = 1e-4f, eps = 1e-8f, dec = 1 - 1e-6f;
    auto bf = [](uint16_t x) { uint32_t u = (uint32_t)x << 16; float f; memcpy(&f, &u, 4); return f; };
    auto tob = [](float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7fffu + ((u >> 16) & 1u)) >> 16); };
    const size_t C = 16384, nc = (n + C - 1) / C;
    for (int rep = 0; rep < 4; ++rep) {
        double t0 = omp_get_wtime();
#pragma omp parallel for schedule(dynamic, 4) num_threads(th)
        for (size_t c = 0; c < nc; ++c) {
            const size_t a = c * C, e = a + C < n ? a + C : n;
#pragma omp simd
            for (size_t i = a; i < e; ++i) {
                const float gf = bf(g[i]);
                const float mi = b1 * m[i] + (1 - b1) * gf, vi = b2 * v[i] + (1 - b2) * gf * gf;
                const float pi = p[i] * dec - lr * mi / (std::sqrt(vi) + eps);
                p[i] = pi; m[i] = mi; v[i] = vi; g[i] = tob(pi);
            }
        }
        double t1 = omp_get_wtime();
#pragma omp parallel for schedule(dynamic, 4) num_threads(th)
        for (size_t c = 0; c < nc; ++c) {
            const size_t a = c * C, e = a + C < n ? a + C : n;
#pragma omp simd
            for (size_t i = a; i < e; ++i) {
                const float gf = bf(g[i]);
                float* r = pmv + 3 * i;
                const float mi = b1 * r[1] + (1 - b1) * gf, vi = b2 * r[2] + (1 - b2) * gf * gf;
                const float pi = r[0] * dec - lr * mi / (std::sqrt(vi) + eps);
                r[0] = pi; r[1] = mi; r[2] = vi; g[i] = tob(pi);
            }
        }
        double t2 = omp_get_wtime();
        printf("threads %d  separate %.1f GB/s  interleaved %.1f GB/s\n", th, 28.0 * n / (t1 - t0) / 1e9, 28.0 * n / (t2 - t1) / 1e9);
    }
}
