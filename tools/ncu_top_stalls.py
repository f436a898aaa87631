"""Top stalled SASS instructions of one kernel launch in an ncu report (source page).

    python tools/ncu_top_stalls.py report.ncu-rep [launch_index] [n]
"""
import csv
import subprocess
import sys


def main(path, launch=0, n=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--launch-skip", str(launch),
                          "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    print(rows[0][1][:120])
    h = rows[1]
    si, ns = h.index("Source"), h.index("# Samples")
    stall = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    data = []
    for idx, r in enumerate(rows[2:]):
        try:
            data.append((int(r[ns]), idx, r[si].strip(), {h[i][6:]: int(r[i]) for i in stall if r[i] not in ("", "0")}))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data)
    print("samples", tot)
    agg = {}
    for d in data:
        for k, v in d[3].items():
            agg[k] = agg.get(k, 0) + v
    print({k: round(100 * v / tot, 1) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])})
    for d in sorted(data, reverse=True)[:n]:
        print(f"{100 * d[0] / tot:5.1f}%  #{d[1]:5d}  {d[2][:70]:70s} {d[3]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 30)
