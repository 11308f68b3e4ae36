"""Per-tile-type throughput from a device timeline trace: tiles completed per 250 us window,
split by task-id range (first GEMM type vs second), plus comm/relay/reduce spans."""
import json, sys
path, n_pre, n_first = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ev = json.load(open(path))["traceEvents"]
t0 = min(e["ts"] for e in ev)
W = 250.0
bins = {}
for e in ev:
    if e["name"] != "comp":
        continue
    t = e["args"]["task"]
    kind = "A" if t < n_pre + n_first else "B"
    b = int((e["ts"] + e["dur"] - t0) // W)
    bins.setdefault(b, {"A": 0, "B": 0})[kind] += 1
for b in sorted(bins):
    print(f"{b*W:7.0f}-{(b+1)*W:7.0f} us  A={bins[b]['A']:5d}  B={bins[b]['B']:5d}")
