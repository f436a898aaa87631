"""Tabulate an `ncu --csv --metrics ...` launch list: one line per launch
(id, kernel, grid, metric values), optionally filtered by a kernel substring."""
import csv
import sys


def main(path, filt=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, im, iv, ig, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Grid Size", "ID"))
    out, names = {}, []
    for r in rows[1:]:
        key = (int(r[ii]), r[ik], r[ig])
        out.setdefault(key, {})[r[im]] = r[iv]
        if r[im] not in names:
            names.append(r[im])
    print("id | kernel | grid | " + " | ".join(names))
    for (i, k, g), v in sorted(out.items()):
        if filt in k:
            print(f"{i} | {k[:70]} | {g} | " + " | ".join(v.get(n, "") for n in names))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
