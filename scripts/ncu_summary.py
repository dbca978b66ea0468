"""Key metrics of every kernel in an ncu report -> JSON lines (for profiles/)."""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_mem_active_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "smsp__inst_executed.sum": "instructions",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")][:90]}
        for k, name in KEYS.items():
            for i, n in enumerate(h):
                if n == k or n.endswith("." + k):
                    d[name] = [r[i], u[i]]
                    break
        print(json.dumps(d))


if __name__ == "__main__":
    main(sys.argv[1])
