"""Warp-stall samples per CUDA source line from an ncu --set full report (source page, cuda,sass):
  python tools/ncu_lines.py report.ncu-rep <launch index> [top N]"""
import collections, csv, io, subprocess, sys

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:megakernel",
                               "--launch-skip", str(idx), "--launch-count", "1", "--print-source", "cuda,sass"],
                              text=True, stderr=subprocess.DEVNULL)
agg = collections.Counter()
agg_ni = collections.Counter()
src = {}
fname, line, cols = "?", "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        cols = r
        continue
    if cols is None or r[0] in ("Function Name",):
        continue
    if r[0]:
        line = r[0]
        src[(fname, line)] = r[1].strip()[:100]
        continue
    try:
        s, ni = int(r[4]), int(r[5])
    except (ValueError, IndexError):
        continue
    agg[(fname, line)] += s
    agg_ni[(fname, line)] += ni
tot = sum(agg.values())
print(f"total samples {tot}")
for key, v in agg.most_common(top):
    print(f"{100.0 * v / tot:5.1f}% {100.0 * agg_ni[key] / tot:5.1f}%  {key[0]}:{key[1]}  {src.get(key, '')}")
if len(sys.argv) > 5:  # file lo hi: every line of a region, in line order
    f, lo, hi = sys.argv[4], int(sys.argv[5]), int(sys.argv[6])
    sub = sorted((int(l), v) for (fn, l), v in agg.items() if fn == f and l.isdigit() and lo <= int(l) <= hi)
    print(f"region {f}:{lo}-{hi}: {100.0 * sum(v for _, v in sub) / tot:.1f}% of samples")
    for l, v in sub:
        print(f"{100.0 * v / tot:5.1f}% {100.0 * agg_ni[(f, str(l))] / tot:5.1f}%  {l}  {src.get((f, str(l)), '')}")
