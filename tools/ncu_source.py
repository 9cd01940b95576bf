"""Per-source-line instruction and stall totals of an ncu report (needs -lineinfo):
    python tools/ncu_source.py gpurun_out/prof.ncu-rep [top]"""
import csv
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    i_src = hdr.index("Source")
    i_ins = hdr.index("Instructions Executed")
    i_smp = hdr.index("Warp Stall Sampling (All Samples)")
    recs = []
    tot_i = tot_s = 0
    for r in rows[2:]:
        if len(r) <= i_ins:
            continue
        try:
            ins = float(r[i_ins] or 0)
            smp = float(r[i_smp] or 0)
        except ValueError:
            continue
        tot_i += ins
        tot_s += smp
        recs.append((smp, ins, r[0], r[i_src].strip()[:110]))
    recs.sort(reverse=True)
    print(f"total instructions {tot_i:.3e}  samples {tot_s:.0f}")
    for smp, ins, line, src in recs[:top]:
        print(f"{100*smp/max(tot_s,1):5.1f}% smp {100*ins/max(tot_i,1):5.1f}% ins  L{line:>5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
