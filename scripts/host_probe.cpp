// Host-side probe for the CpuOptim lane (measurement tool, not product code): host DRAM
// bandwidth of the in-place 28 B/param pattern (fp32 p/m/v read+write, bf16 g read + bf16 out
// write) with trivial arithmetic ("stream") versus the real host AdamW (ah_cpu_adam), for
// several thread counts and three ways of obtaining pinned memory:
//   cuda   cudaHostAlloc (what the executor uses today)
//   thp    2 MiB-aligned malloc + madvise(MADV_HUGEPAGE) + cudaHostRegister
//   plain  4 KiB pages + cudaHostRegister
// Build on the box: g++ -O3 -march=native -fopenmp scripts/host_probe.cpp -I include
//   -I/usr/local/cuda/include -L paper_2503_01890_b200/lib -lautohete -L/usr/local/cuda/lib64 -lcudart
#include <cuda_runtime.h>
#include <omp.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "autohete.h"

static void* get(const char* kind, size_t bytes) {
    void* p = nullptr;
    if (!strcmp(kind, "cuda")) {
        if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) return nullptr;
        return p;
    }
    const size_t a = 2u << 20;
    bytes = (bytes + a - 1) / a * a;
    if (posix_memalign(&p, a, bytes)) return nullptr;
    if (!strcmp(kind, "thp")) madvise(p, bytes, MADV_HUGEPAGE);
    else madvise(p, bytes, MADV_NOHUGEPAGE);
    memset(p, 0, bytes);
    if (cudaHostRegister(p, bytes, cudaHostRegisterPortable) != cudaSuccess) return nullptr;
    return p;
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 200000000ull;
    const char* kinds[] = {"cuda", "thp", "plain"};
    for (const char* kind : kinds) {
        float* p = (float*)get(kind, n * 4);
        float* m = (float*)get(kind, n * 4);
        float* v = (float*)get(kind, n * 4);
        uint16_t* g = (uint16_t*)get(kind, n * 2);
        if (!p || !m || !v || !g) { printf("{\"alloc\":\"%s\",\"error\":\"alloc failed\"}\n", kind); continue; }
#pragma omp parallel for
        for (size_t i = 0; i < n; ++i) { p[i] = 0.01f; m[i] = 0.f; v[i] = 0.f; g[i] = 0x3c00; }
        ah_adam_hparams hp{1e-4f, 0.9f, 0.999f, 1e-8f, 0.01f, 3};
        for (int t : {1, 8, 12, 14, 16}) {
            double best_s = 1e9, best_a = 1e9;
            for (int r = 0; r < 4; ++r) {
                auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(t) schedule(static)
                for (size_t i = 0; i < n; ++i) {
                    p[i] *= 0.999f; m[i] *= 0.999f; v[i] *= 0.999f; g[i] ^= 1;
                }
                auto t1 = std::chrono::steady_clock::now();
                ah_cpu_adam(&hp, p, m, v, g, g, n, 1.f, t);
                auto t2 = std::chrono::steady_clock::now();
                if (r) {
                    best_s = std::min(best_s, std::chrono::duration<double>(t1 - t0).count());
                    best_a = std::min(best_a, std::chrono::duration<double>(t2 - t1).count());
                }
            }
            printf("{\"alloc\":\"%s\",\"threads\":%d,\"stream_GBps\":%.1f,\"adam_GBps\":%.1f,\"adam_Gparams\":%.3f}\n",
                   kind, t, 28.0 * n / best_s / 1e9, 28.0 * n / best_a / 1e9, n / best_a / 1e9);
            fflush(stdout);
        }
        {  // host-link DMA from this kind of pinned memory (1.6 GB of the fp32 buffer p)
            const size_t bytes = std::min(n * 4, (size_t)1600 << 20);
            void* d = nullptr;
            cudaMalloc(&d, bytes);
            cudaStream_t st;
            cudaStreamCreate(&st);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best_h = 1e9, best_d = 1e9;
            for (int r = 0; r < 4; ++r) {
                float ms;
                cudaEventRecord(e0, st);
                cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, st);
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                if (r) best_h = std::min(best_h, ms);
                cudaEventRecord(e0, st);
                cudaMemcpyAsync(p, d, bytes, cudaMemcpyDeviceToHost, st);
                cudaEventRecord(e1, st);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                if (r) best_d = std::min(best_d, ms);
            }
            printf("{\"alloc\":\"%s\",\"h2d_GBps\":%.1f,\"d2h_GBps\":%.1f}\n", kind, bytes / best_h / 1e6,
                   bytes / best_d / 1e6);
            cudaFree(d);
        }
        if (!strcmp(kind, "cuda")) { cudaFreeHost(p); cudaFreeHost(m); cudaFreeHost(v); cudaFreeHost(g); }
        else { for (void* x : {(void*)p, (void*)m, (void*)v, (void*)g}) { cudaHostUnregister(x); free(x); } }
    }
    return 0;
}
