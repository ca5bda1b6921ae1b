"""Per-source-line attribution of an ncu report (instructions executed, stall samples):
python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f = None
    h = None
    inst, smp, src = collections.Counter(), collections.Counter(), {}
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            h = r
            ie, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
            continue
        if h is None or len(r) < len(h) or not r[0]:
            continue
        k = (f, int(r[0]))
        src[k] = r[1].strip()[:90]
        try:
            inst[k] += int(r[ie] or 0)
            smp[k] += int(r[iss] or 0)
        except ValueError:
            pass
    ti, ts = sum(inst.values()), sum(smp.values())
    print(f"instructions executed {ti:,}  stall samples {ts:,}")
    print("-- by instructions")
    for k, v in inst.most_common(top):
        print(f"{v / ti * 100:5.1f}% inst {smp[k] / ts * 100:5.1f}% smp  {k[0]}:{k[1]}: {src[k]}")
    print("-- by stall samples")
    for k, v in smp.most_common(top // 2):
        print(f"{inst[k] / ti * 100:5.1f}% inst {v / ts * 100:5.1f}% smp  {k[0]}:{k[1]}: {src[k]}")


if __name__ == "__main__":
    main()
