"""Top SASS instructions by warp-stall samples from an ncu report (source page, SASS view).
    python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ai, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
def num(v):
    try:
        return float(v)
    except ValueError:
        return None


data = [r for r in rows[2:] if len(r) > si and num(r[si]) is not None]
tot = sum(num(r[si]) for r in data)
print(f"total samples {tot:.0f}")
for idx, r in sorted(enumerate(data), key=lambda x: -num(x[1][si]))[:top]:
    print(f"{idx:5d} {num(r[si]):7.0f} {100*num(r[si])/tot:5.1f}%  {r[ai].strip()[:80]}")
