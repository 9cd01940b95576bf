"""Per-source-line instruction and stall totals of an ncu report (needs -lineinfo):
    python tools/ncu_source.py gpurun_out/prof.ncu-rep [top]"""
import csv
import os
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    recs = []
    tot_i = tot_s = 0.0
    fname, hdr = "?", None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Line No":
            hdr = r
            i_ins = hdr.index("Instructions Executed")
            i_smp = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or not r[0].isdigit() or len(r) <= i_ins or r[2] != "-":
            continue
        try:
            ins = float(r[i_ins] or 0)
            smp = float(r[i_smp] or 0)
        except ValueError:
            continue
        tot_i += ins
        tot_s += smp
        recs.append((smp, ins, f"{fname}:{r[0]}", r[1].strip()[:100]))
    recs.sort(reverse=True)
    print(f"total instructions {tot_i:.3e}  samples {tot_s:.0f}")
    for smp, ins, loc, src in recs[:top]:
        print(f"{100 * smp / max(tot_s, 1):5.1f}% smp {100 * ins / max(tot_i, 1):5.1f}% ins "
              f"{loc:24s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
