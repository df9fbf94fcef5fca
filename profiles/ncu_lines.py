"""Per-source-line hotspots of an ncu report captured with -lineinfo and
--import-source on (run here, no GPU needed):
    python profiles/ncu_lines.py gpurun_out/x.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    cur, agg = None, []
    for r in csv.reader(out.splitlines()):
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
        elif len(r) > 8 and r[0].isdigit():
            try:
                samp, inst = int(r[4]), int(r[7])
            except ValueError:
                continue
            if samp or inst:
                agg.append((samp, inst, f"{cur}:{r[0]}", r[1].strip()[:80]))
    ts, ti = sum(a[0] for a in agg), sum(a[1] for a in agg)
    print(f"stall samples {ts}, warp instructions {ti}")
    for s, i, loc, src in sorted(agg, reverse=True)[:top]:
        print(f"{100 * s / max(ts, 1):5.1f}% {100 * i / max(ti, 1):5.1f}%  {loc:24s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
