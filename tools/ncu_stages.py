"""Per-kernel summary of an ncu --set full report: duration, DMMA sub-pipe
busy %, DRAM bytes, L2 hit rate, registers (the numbers profiles/ quotes)."""
import csv
import json
import subprocess
import sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "dmma_pipe_active_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_hit_rate_pct": "lts__t_sector_hit_rate.pct",
    "registers_per_thread": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k, m in KEYS.items():
            if m in h:
                i = h.index(m)
                v = float(r[i].replace(",", "")) if r[i] else None
                u = units[i]
                if v is not None and u == "Gbyte":
                    v *= 1e9
                elif v is not None and u == "Mbyte":
                    v *= 1e6
                elif v is not None and u == "usecond":
                    v /= 1e3
                d[k] = v
        res.append(d)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
