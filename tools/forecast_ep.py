"""B200 perf-model forecast (predict_layer with the round-2 calibration) of the EP=2/4/8 scaling configs:
weak scaling, 16K tokens per GPU, choose_config()'s launch parameters, NVLink at 770 GB/s per direction
(and the 900 GB/s spec). Writes a markdown table; the driver's 8-GPU run is what checks it.
  python tools/forecast_ep.py > profiles/r02_model_forecast_ep.md
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_19241_b200 import model as Mo  # noqa: E402


def main():
    peaks = json.load(open(os.path.join(bench.ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(bench.ROOT, "MEASURED_PEAKS.json")) else {}
    p_peak = peaks.get("bf16_tflops_sustained", 1408.1) * 1e12
    bw_hbm = peaks.get("hbm_gbs", 6468.9) * 1e9
    print("# B200 perf-model forecast (predict_layer, round-2 calibration: 94 measured cases incl. 18 virtual-rank")
    print("# EP=2/4/8 cases, profiles/r02_perf_model_validation.md) for the EP=2/4/8 scaling configs -- weak scaling,")
    print(f"# 16K tokens per GPU, choose_config()'s launch parameters, P = {p_peak / 1e12:.1f} TFLOP/s sustained,")
    print(f"# HBM {bw_hbm / 1e9:.0f} GB/s. ms per fwd+bwd step per GPU; tokens/s aggregate over the EP GPUs. To be checked")
    print("# against the driver's 8-GPU run (tools/scale_run.sh).")
    print("| config | EP | n_disp | n_relay | fwd disp | fwd comb | bwd disp | bwd comb | step ms | t_gemm | "
          "t_nvl 770 | step ms @900 | tokens/s (all GPUs) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name in ("mixtral", "qwen3", "dsv3"):
        H, F, E, k, T = bench.CONFIGS[name]
        for ep in (1, 2, 4, 8):
            cfg = Mo.choose_config(H, F, E, k, T, ep)
            s = Mo.shape(H, F, E, k, T)
            p = Mo.predict_layer(s, Mo.hw(ep, p_peak=p_peak, bw_hbm=bw_hbm), cfg)
            p9 = Mo.predict_layer(s, Mo.hw(ep, p_peak=p_peak, bw_hbm=bw_hbm, bw_nvl=900e9), cfg)
            print(f"| {name} | {ep} | {cfg.n_disp} | {cfg.n_relay} | {p.fwd_dispatch * 1e3:.2f} | "
                  f"{p.fwd_combine * 1e3:.2f} | {p.bwd_dispatch * 1e3:.2f} | {p.bwd_combine * 1e3:.2f} | "
                  f"{p.total * 1e3:.2f} | {p.t_gemm_bound * 1e3:.2f} | {p.t_nvl_bound * 1e3:.2f} | "
                  f"{p9.total * 1e3:.2f} | {T * ep / p.total:,.0f} |")


if __name__ == "__main__":
    main()
