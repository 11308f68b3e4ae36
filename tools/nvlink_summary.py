"""Summarise tools/ncu_nvlink.sh: per MegaKernel, NVLink TX/RX bytes per rank (ncu) and GB/s per
direction over the kernel's unprofiled duration (bench.py kernel_ms), against 770 GB/s measured /
900 GB/s nominal per direction."""
import csv
import io
import json
import sys

KIND = {"0, ModeUp": "fwd_dispatch_gemm(+plan)", "1, ModeDown": "fwd_gemm_combine",
        "2, ModeDgradDown": "bwd_dispatch_gemm", "3, ModeDgradUp": "bwd_gemm_combine"}
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
bench = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
kms = bench["kernel_ms"]
acc = {}
for r in csv.DictReader(io.StringIO(txt)):
    n = r["Kernel Name"]
    n = n.split("<")[1].split(">")[0] if "<" in n else n
    key = (r["Process ID"], KIND.get(n, n))
    acc.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
print(f"# NVLink per MegaKernel, EP={bench['n_gpus']}, {bench['config']['workload']}")
print("| rank (pid) | kernel | TX GB | RX GB | ms (unprofiled) | TX GB/s | RX GB/s | TX / 900 |")
print("|---|---|---|---|---|---|---|---|")
for (pid, k), m in sorted(acc.items()):
    ms = kms.get(k)
    tx, rx = m.get("nvltx__bytes.sum", 0) / 1e9, m.get("nvlrx__bytes.sum", 0) / 1e9
    if ms:
        print(f"| {pid} | {k} | {tx:.3f} | {rx:.3f} | {ms:.3f} | {tx / ms * 1e3:.0f} | {rx / ms * 1e3:.0f} | "
              f"{tx / ms * 1e3 / 900:.2f} |")
