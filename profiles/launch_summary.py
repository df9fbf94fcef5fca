"""Summarise an ncu launch list (gpu__time_duration.sum CSV) into the kernels of
the last decision round:  python profiles/launch_summary.py launches.csv out.txt "cmd" """
import csv
import sys


def main(src, dst, cmd):
    rows = list(csv.reader(open(src)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.append((d["Kernel Name"], float(d["Metric Value"])))
    idx = [i for i, (n, _) in enumerate(out) if "k_horizon_divergence" in n]
    last = out[idx[-1]:]
    # one round: up to the ordered S_e (later launches belong to the next timing)
    ends = [i for i, (n, _) in enumerate(last) if "k_small_apply" in n] or \
        [i for i, (n, _) in enumerate(last) if "k_run_merge" in n]
    if ends:
        last = last[:ends[0] + 1]
    tot = sum(v for _, v in last)
    with open(dst, "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n")
        f.write(f"# command: {cmd}\n# one decision round (last in the run); total {tot / 1e3:.1f} us\n")
        for n, v in last:
            f.write(f"{v / 1e3:10.1f} us  {100 * v / tot:5.1f}%  {n[:110]}\n")
    print(open(dst).read())


if __name__ == "__main__":
    main(*sys.argv[1:4])
