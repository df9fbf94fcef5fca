"""Per-kernel table (time + DRAM bytes) of the last decision round in an ncu
launch list taken with --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv:
    python profiles/launch_table.py launches.csv out.txt "command" [kernels_per_round]"""
import csv
import sys
from collections import OrderedDict


def main(src, dst, cmd, per_round=0):
    rows = list(csv.reader(open(src)))
    hdr, d = None, OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            i = int(r[hdr.index("ID")])
            d.setdefault(i, {"name": r[hdr.index("Kernel Name")]})[r[hdr.index("Metric Name")]] = \
                float(r[hdr.index("Metric Value")].replace(",", ""))
    ids = [i for i in d if "kr::" in d[i]["name"]]
    if per_round <= 0:  # the kernels after the last horizon launch (one round)
        last = max(i for i in ids if "k_horizon" in d[i]["name"])
        ids = [i for i in ids if i >= last]
    else:
        ids = ids[-per_round:]
    lines = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
             "--clock-control none (cold cache, serialised)", f"# command: {cmd}",
             "#   time_us   dram_MB    GB/s  kernel"]
    tt = tb = 0.0
    for i in ids:
        m = d[i]
        t = m.get("gpu__time_duration.sum", 0) / 1e3
        b = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
        tt += t
        tb += b
        lines.append(f"{t:10.1f} {b:9.1f} {1e3 * b / t if t else 0:7.0f}  {m['name'][:110]}")
    lines.append(f"# total {tt:.1f} us, {tb:.0f} MB (serialised; the round overlaps the side stream)")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0)
