"""SASS-level hot spots of an ncu report: top instructions by stall samples and
the executed-instruction mix by opcode.
    python tools/ncu_sass.py gpurun_out/prof.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys


def main(path, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    i_src, i_ins = hdr.index("Source"), hdr.index("Instructions Executed")
    i_smp = hdr.index("Warp Stall Sampling (All Samples)")
    recs, mix = [], collections.Counter()
    tot_i = tot_s = 0
    for idx, r in enumerate(rows[2:]):
        try:
            ins, smp = float(r[i_ins] or 0), float(r[i_smp] or 0)
        except (ValueError, IndexError):
            continue
        op = r[i_src].split()[0] if r[i_src].split() else "?"
        if op.startswith("@"):
            op = r[i_src].split()[1]
        mix[op.split(".")[0]] += ins
        tot_i += ins
        tot_s += smp
        recs.append((smp, ins, idx, r[i_src].strip()[:90]))
    print(f"total instructions {tot_i:.4e} samples {tot_s:.0f}")
    for op, n in mix.most_common(18):
        print(f"  {op:10s} {100*n/tot_i:5.1f}%")
    for smp, ins, idx, src in sorted(recs, reverse=True)[:top]:
        print(f"{100*smp/tot_s:5.1f}% smp {ins:10.0f} ins  #{idx:<5} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
