/* hetsim_c.h — extern "C" view of the drop-in hetsim::core planner / scheduler, for hosts that
 * bind C (ctypes, cgo, JNI). Each call mirrors a reference library entry
 * (proj/README.md:182-192 library usage; proj/tools/hetsim_main.cpp:77-130 plan_and_tune /
 * cmd_plan); exceptions become negative return codes + ah_hetsim_last_error().
 * Implemented in libhetsim_core.so (paper_2503_01890_b200/csrc/hetsim/c_api.cpp). */
#ifndef HETSIM_C_H
#define HETSIM_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HETSIM_OK 0
#define HETSIM_ERR_CONFIG -1     /* hetsim::ConfigError (config.hpp:13) */
#define HETSIM_ERR_INVALID -2    /* std::invalid_argument */
#define HETSIM_ERR_INFEASIBLE -3 /* hetsim::InfeasibleError (planner.hpp:35) */
#define HETSIM_ERR_MEMORY -4     /* hetsim::MemoryExceededError (simulator.hpp:117) */
#define HETSIM_ERR_OTHER -5

const char* ah_hetsim_last_error(void);

/* block_param_count (workload.hpp:100 / workload.cpp:41-44) */
int64_t ah_hetsim_block_param_count(int64_t hidden_size);

/* `hetsim plan CONFIG` without the file system (hetsim_main.cpp:92-130): parse the INI text,
 * build_profile -> solve -> fine_tune_prefetch, then write_plan_json into out (NUL-terminated).
 * Returns the JSON length + 1 on success (call with out=NULL to size), < 0 on error. */
int64_t ah_hetsim_plan_json(const char* config_text, char* out, size_t cap);

/* Data-parallel extension (hetsim/dp_planner.hpp, not in the reference): plan for dp_size ranks
 * with per-rank sharded optimizer state; collective_gbps <= 0 leaves collectives unmodelled.
 * dp_size == 1 returns exactly ah_hetsim_plan_json's document. */
int64_t ah_hetsim_plan_dp_json(const char* config_text, int32_t dp_size, double collective_gbps, char* out,
                               size_t cap);

/* `hetsim simulate CONFIG` (hetsim_main.cpp:132-201): plan (or use the given strategy when
 * c_hat >= 0), run(n_iters, priority) and write the Chrome trace (simulator.cpp:598-613). */
int64_t ah_hetsim_simulate_trace(const char* config_text, int32_t c_hat, int32_t p_hat, int32_t o_hat,
                                 int32_t n_iters, int32_t priority, char* out, size_t cap);

#ifdef __cplusplus
}
#endif

#endif /* HETSIM_C_H */
