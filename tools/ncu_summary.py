"""Summarise ncu outputs into profiles/: the launch list (--metrics gpu__time_duration.sum) and a
--set full capture of the four MegaKernels (tensor pipe, SM throughput, DRAM traffic, L2 hit, clock).
  python tools/ncu_summary.py launches gpurun_out/launches_mixtral.csv profiles/<name>.txt
  python tools/ncu_summary.py full gpurun_out/prof_mixtral.ncu-rep profiles/<name>.md <config> [traffic.json]"""
import collections, csv, io, json, subprocess, sys

mode = sys.argv[1]
if mode == "launches":
    rows = [r for r in csv.reader(open(sys.argv[2])) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    tot = 0.0
    for r in rows:
        name = r[4][:70]
        v = float(r[-1])
        tot += v
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    with open(sys.argv[3], "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 "
                "--no-cpu-baseline\n# kernel, launches, total, share of all GPU time in the run (warm-up, the "
                "per-kernel pass, the graph replays, the timeline step and the e2e steps included)\n")
        for n, (c, v) in agg.items():
            f.write(f"{n:70s} n={c:3d} total={v / 1e6:9.3f} ms share={100 * v / tot:5.1f}%\n")
    print(open(sys.argv[3]).read())
else:
    raw = subprocess.check_output(["ncu", "-i", sys.argv[2], "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    g = lambda d, w: d[hdr.index(w)]
    names = {"0": "fwd_dispatch_gemm", "1": "fwd_gemm_combine", "2": "bwd_dispatch_gemm", "3": "bwd_gemm_combine"}
    cfg = sys.argv[4]
    lines = [f"# ncu --set full --clock-control none -k regex:megakernel -s 4 -c 4 (tools/step_profile.py --ncu "
             f"--config {cfg}: 1 warm-up + 1 EP=1 step). ncu serialises kernels and replays each ~40x: compare "
             "shares, not absolutes.",
             "| kernel | duration | tensor pipe active | SM throughput | DRAM read | DRAM write | DRAM % of peak | "
             "L2 hit | SM clock | regs |", "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for d in data:
        kn = g(d, "Kernel Name")
        nm = names[kn.split("<")[1].split(",")[0]]
        rd = float(g(d, "dram__bytes_read.sum")) * 1e9
        wr = float(g(d, "dram__bytes_write.sum")) * 1e9
        traffic[f"{cfg}:{nm}"] = rd + wr
        lines.append(
            f"| {nm} | {g(d, 'gpu__time_duration.sum')} ms | "
            f"{float(g(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active')):.1f} % | "
            f"{float(g(d, 'sm__throughput.avg.pct_of_peak_sustained_elapsed')):.1f} % | {rd / 1e9:.2f} GB | "
            f"{wr / 1e9:.2f} GB | {float(g(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')):.1f} % | "
            f"{float(g(d, 'lts__t_sector_hit_rate.pct')):.1f} % | "
            f"{float(g(d, 'sm__cycles_elapsed.avg.per_second')):.3f} GHz | {g(d, 'launch__registers_per_thread')} |")
    open(sys.argv[3], "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if len(sys.argv) > 5:
        t = json.load(open(sys.argv[5]))
        t.update(traffic)
        json.dump(t, open(sys.argv[5], "w"), indent=1)
