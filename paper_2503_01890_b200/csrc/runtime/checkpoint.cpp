// Optimizer-state checkpoint / resume for the executor (the reference has
// only plan persistence, proj/core/src/plan_io.cpp:44-89).
//
// Layout (little-endian): "AHCKPT01", int32 {L, h, nh, s, B, V, dp_rank, dp_size, step},
// int64 per-block element count, then for block 1..L: master | m | v (fp32, this rank's shard or
// the whole block), then wte, wpe, lnf: master | m | v. Where each block's state lives (GPU or
// pinned host) is a property of the plan, not of the file, so a checkpoint moves between plans.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "executor.h"
#include "../kernels/kernels.h"

namespace ah {

struct CheckpointIO {
    static void xfer(Trainer& t, float* state, bool host, size_t n, std::FILE* f, bool write) {
        std::vector<float> buf(n);
        if (write) {
            if (host)
                std::memcpy(buf.data(), state, n * 4);
            else
                t.check(cudaMemcpy(buf.data(), state, n * 4, cudaMemcpyDeviceToHost), "checkpoint d2h");
            if (std::fwrite(buf.data(), 4, n, f) != n) throw std::runtime_error("checkpoint: short write");
        } else {
            if (std::fread(buf.data(), 4, n, f) != n) throw std::runtime_error("checkpoint: short read");
            if (host)
                std::memcpy(state, buf.data(), n * 4);
            else
                t.check(cudaMemcpy(state, buf.data(), n * 4, cudaMemcpyHostToDevice), "checkpoint h2d");
        }
    }

    static void run(Trainer& t, const std::string& path, bool write) {
        t.drain();
        std::FILE* f = std::fopen(path.c_str(), write ? "wb" : "rb");
        if (!f) throw std::runtime_error("checkpoint: cannot open " + path);
        const GptDims& d = t.d_;
        int32_t hdr[9] = {d.L, d.h, d.nh, d.s, d.B, d.V, t.dp_rank_, t.dp_size_, t.step_base_ + (int)t.submitted_};
        const int64_t per_block = (int64_t)(t.dp_ ? t.shard_ : d.m_p());
        char magic[8] = {'A', 'H', 'C', 'K', 'P', 'T', '0', '1'};
        try {
            if (write) {
                std::fwrite(magic, 1, 8, f);
                std::fwrite(hdr, 4, 9, f);
                std::fwrite(&per_block, 8, 1, f);
            } else {
                char m2[8];
                int32_t h2[9];
                int64_t pb = 0;
                if (std::fread(m2, 1, 8, f) != 8 || std::memcmp(m2, magic, 8) != 0)
                    throw std::runtime_error("checkpoint: bad magic");
                if (std::fread(h2, 4, 9, f) != 9 || std::fread(&pb, 8, 1, f) != 1)
                    throw std::runtime_error("checkpoint: truncated header");
                // shape + dp layout; the batch size (hdr[4]) does not enter the optimizer state
                const int cmp[7] = {0, 1, 2, 3, 5, 6, 7};
                bool same = pb == per_block;
                for (int c : cmp) same = same && h2[c] == hdr[c];
                if (!same)
                    throw std::invalid_argument("checkpoint: model shape / data-parallel layout mismatch");
                if (t.submitted_ != 0) throw std::logic_error("checkpoint: load before the first iteration");
                t.step_base_ = h2[8];
            }
            for (int i = 1; i <= d.L; ++i) {
                Trainer::BlockState& b = t.blocks_[(size_t)i];
                for (float* p : {b.master, b.m1, b.m2}) xfer(t, p, b.o, (size_t)per_block, f, write);
                if (!write && b.o) {  // refresh the host bf16 copy the next prefetch sends up
                    std::vector<uint16_t> tmp((size_t)per_block);
                    for (size_t k = 0; k < (size_t)per_block; ++k) {
                        uint32_t u;
                        std::memcpy(&u, &b.master[k], 4);
                        const uint32_t rne = (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
                        tmp[k] = (uint16_t)(((u & 0x7fffffffu) > 0x7f800000u) ? ((u >> 16) | 0x40u) : rne);
                    }
                    std::memcpy(b.host_bf16, tmp.data(), tmp.size() * 2);
                }
            }
            const size_t nwte = (size_t)d.Vp * d.h, nwpe = (size_t)d.s * d.h, nlnf = 2 * (size_t)d.h;
            const std::pair<float*, size_t> emb[9] = {{t.wte_, nwte}, {t.wte_m_, nwte}, {t.wte_v_, nwte},
                                                      {t.wpe_, nwpe}, {t.wpe_m_, nwpe}, {t.wpe_v_, nwpe},
                                                      {t.lnf_, nlnf}, {t.lnf_m_, nlnf}, {t.lnf_v_, nlnf}};
            for (const auto& e : emb) xfer(t, e.first, false, e.second, f, write);
            if (!write) {  // bf16 working copies of the replicated parameters
                t.check(launch_cast_f32_bf16(t.wte_, t.wte_b_, nwte, t.s_compute_), "cast");
                t.check(launch_cast_f32_bf16(t.wpe_, t.wpe_b_, nwpe, t.s_compute_), "cast");
                t.check(launch_cast_f32_bf16(t.lnf_, t.lnf_b_, nlnf, t.s_compute_), "cast");
                t.check(cudaStreamSynchronize(t.s_compute_), "sync");
            }
        } catch (...) {
            std::fclose(f);
            throw;
        }
        std::fclose(f);
    }
};

void Trainer::save(const std::string& path) { CheckpointIO::run(*this, path, true); }
void Trainer::load(const std::string& path) { CheckpointIO::run(*this, path, false); }

}  // namespace ah
