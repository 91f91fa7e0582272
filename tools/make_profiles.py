"""Write the committed evidence under profiles/ from one gpu_full.sh run.

    python tools/make_profiles.py TAG [ROUND]

Reads gpurun_out/{bench,bench_ref,sweep,stack,launches,prof,prof_b8}_TAG.* and writes
profiles/rNN_bench.json, rNN_bench_ref.json, rNN_sweep.md, rNN_stack_tp1.json,
rNN_launches_fc1.csv, rNN_ncu_fc1.md and profiles/ncu_summary.json (read by bench.py for
roofline.traffic).
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
sys.path.insert(0, ROOT)
from bench import algorithmic_bytes  # noqa: E402

SM_HZ = 1.965e9


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(d, k, scale=1.0):
    v, u = d[k]
    f = float(v.replace(",", ""))
    mult = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}.get(u, 1.0)
    return f * mult * scale


def stalls(d):
    import re
    st = []
    for k, (v, _) in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(.*)_per_issue_active.ratio", k)
        if m:
            try:
                st.append((float(v), m.group(1)))
            except ValueError:
                pass
    return sorted(st, reverse=True)[:6]


def main(tag, rnd="01"):
    p = lambda f: os.path.join(OUT, f)  # noqa: E731
    bench = json.loads(open(p(f"bench_{tag}.json")).read().strip().splitlines()[-1])
    ref = json.loads(open(p(f"bench_ref_{tag}.json")).read().strip().splitlines()[-1])
    json.dump(bench, open(os.path.join(PROF, f"r{rnd}_bench.json"), "w"), indent=1)
    json.dump(ref, open(os.path.join(PROF, f"r{rnd}_bench_ref.json"), "w"), indent=1)
    shutil.copy(p(f"launches_{tag}.csv"), os.path.join(PROF, f"r{rnd}_launches_fc1.csv"))
    stack = json.loads(open(p(f"stack_{tag}.json")).read().strip().splitlines()[-1])
    json.dump(stack, open(os.path.join(PROF, f"r{rnd}_stack_tp1.json"), "w"), indent=1)

    # launch list summary
    rows = [r for r in csv.reader(l for l in open(p(f"launches_{tag}.csv")) if not l.startswith("=="))]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    per = {}
    for r in rows[1:]:
        try:
            per.setdefault(r[ik].split("(")[0], []).append(float(r[iv].replace(",", "")) / 1e3)
        except (ValueError, IndexError):
            pass

    B = algorithmic_bytes(49152, 12288, 3, 128)
    g = raw(p(f"prof_{tag}.ncu-rep"))
    b8 = raw(p(f"prof_b8_{tag}.ncu-rep"))
    gname = g["Kernel Name"][0]
    bname = b8["Kernel Name"][0]
    rd, wr = num(g, "dram__bytes_read.sum"), num(g, "dram__bytes_write.sum")
    summ = {
        "lut_gemv_kernel": {
            "kernel": f"{gname} fused mode (fc1: m=49152, n=12288, q=3, g=128, b=1; 144 CTAs = 12 slices x 12)",
            "source": f"ncu --set full --clock-control none -k regex:lut_gemv -s 10 -c 1 (profiles/r{rnd}_ncu_fc1.md), tag {tag}",
            "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
            "algorithmic_bytes": B, "ncu_duration_us": round(num(g, "gpu__time_duration.sum"), 3),
            "inst_executed": int(num(g, "smsp__inst_executed.sum")),
            "shared_ld_inst": int(num(g, "smsp__sass_inst_executed_op_shared_ld.sum")),
            "shared_ld_bank_conflicts": int(num(g, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")),
            "shared_wavefronts": int(num(g, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")),
            "issue_active_pct": round(num(g, "smsp__issue_active.avg.pct_of_peak_sustained_active"), 2),
            "lsu_pipe_pct": round(num(g, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"), 2),
        },
        "batched_b8_kernel": {
            # b = 8 runs as two b = 4 chunks (batch split): the capture is one chunk's lut_gemvv_kernel
            "kernel": f"{bname} (fc1, b=8: one of its two b=4 chunks)",
            "source": f"ncu --set full --clock-control none -k regex:lut_gemvv -s 1 -c 1, tag {tag}",
            "dram_bytes_per_launch": int(num(b8, "dram__bytes_read.sum") + num(b8, "dram__bytes_write.sum")),
            "algorithmic_bytes": algorithmic_bytes(49152, 12288, 3, 128, 4),
            "ncu_duration_us": round(num(b8, "gpu__time_duration.sum"), 3),
            "shared_wavefronts": int(num(b8, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")),
            "shared_ld_bank_conflicts": int(num(b8, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum")),
            "lookups": 49152 * 3 * (12288 // 8) * 8,
        },
    }
    json.dump(summ, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)

    lines = [f"# Round {int(rnd)} -- ncu evidence for the LUT-GEMM GEMV (fc1, q=3, g=128, b=1), tag {tag}", "",
             "Workload: OPT-175B FFN-1, W is 49152 x 12288 (out x in), q=3, g=128, b=1.",
             f"Algorithmic bytes B_alg = m n q/8 + 2 m (n/g) q + 2n + 2m = {B:,} B (SURVEY 8(d)).", "",
             "## Launch list of the bench command (`ncu --metrics gpu__time_duration.sum --clock-control none`,"
             " eager, serialized, cold L2)", "",
             f"File: `r{rnd}_launches_fc1.csv`.", "", "| kernel | launches | mean us |", "|---|---|---|"]
    for k, v in per.items():
        lines.append(f"| `{k.split('::')[-1]}` | {len(v)} | {sum(v) / len(v):.2f} |")
    tot = sum(sum(v) for k, v in per.items() if "lut_" in k)
    gem = sum(sum(v) for k, v in per.items() if "lut_gemv" in k)
    lines += ["", f"`lut_gemv_kernel` share of the product kernels' time: {100 * gem / max(tot, 1e-9):.1f} % "
              "(one launch per GEMV: the cross-slice reduction is fused). Pack kernels are offline.", "",
              f"In the timed bench (CUDA graph of consecutive GEMVs): {bench['us_per_gemv']} us per GEMV, "
              f"{bench['value']} GB/s = {100 * bench['roofline']['frac']:.1f} % of the measured "
              f"{bench['roofline']['peak']} GB/s (this box's copy: {bench['roofline'].get('box_copy_gbs')} GB/s).",
              "", f"## One LUT kernel, `ncu --set full --clock-control none --import-source on` ({gname})", "",
              "| metric | value |", "|---|---|"]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__cycles_active.avg",
            "sm__cycles_elapsed.avg"]
    for k in keys:
        if k in g:
            lines.append(f"| {k} | {g[k][0]} {g[k][1]} |")
    lines += [f"| traffic / B_alg | {(rd + wr) / B:.3f} |",
              f"| stalls (cycles per issued instr.) | {', '.join(f'{n} {v:.2f}' for v, n in stalls(g))} |", "",
              f"## One batched kernel (fc1, b=8), `ncu --set full` ({bname})", "", "| metric | value |", "|---|---|"]
    for k in keys:
        if k in b8:
            lines.append(f"| {k} | {b8[k][0]} {b8[k][1]} |")
    lk = 49152 * 3 * (12288 // 8) * 8
    lines += [f"| lookups | {lk:,} (= {lk // 32:,} warp-lookups of 4 B, i.e. fp32 LUT bytes / 128 per wavefront) |",
              f"| stalls | {', '.join(f'{n} {v:.2f}' for v, n in stalls(b8))} |", ""]
    open(os.path.join(PROF, f"r{rnd}_ncu_fc1.md"), "w").write("\n".join(lines) + "\n")

    # sweep table
    allsw = [json.loads(l) for l in open(p(f"sweep_{tag}.jsonl")) if l.strip().startswith("{")]
    sw = [d for d in allsw if not d["case"].startswith(("dense", "quantize"))]
    quant = [d for d in allsw if d["case"].startswith("quantize")]
    dense = {d["b"]: d for d in allsw if d["case"].startswith("dense")}
    t = [f"# Round {int(rnd)} -- all BASELINE shapes (tools/sweep.py, CUDA-graph timing, B200), tag {tag}", "",
         "Timing: CUDA graph of consecutive products on rotating weight copies (> 3x L2), events around the replays;"
         " us per product. Peak = measured 6544.7 GB/s (`MEASURED_PEAKS.json`). LDS roof = fp32 LUT bytes /"
         " (128 B/clk/SM x 148 SMs x 1.965 GHz).", "", "## b = 1 (GEMV)", "",
         "| case | m | n | q | g | offset | compact | compression vs fp16 | us | GB/s | % of HBM peak | HBM roof us |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in sw:
        if d["b"] == 1:
            cr = 2 * d["m"] * d["n"] / (d["bytes_alg"] - 2 * d["n"] - 2 * d["m"])
            t.append(f"| {d['case']} | {d['m']} | {d['n']} | {d['q']} | {d['g']} | {d['offset']} | "
                     f"{d.get('compact', False)} | {cr:.2f}x | {d['us']} | {d['GBps']} | {100 * d['frac_hbm']:.1f} | "
                     f"{d['hbm_roof_us']} |")
    att = sorted([d for d in sw if d["case"].startswith("attn_")], key=lambda d: d["bytes_alg"])
    if att:
        t += ["", "Latency vs compression ratio on the 12288 x 12288 layer (the analogue of Fig. 4(b), P:L309-313: "
              "for batch 1 the latency follows the memory footprint; (q, g) pairs of similar footprint take "
              "similar time):", "", "| q | g | compression vs fp16 | MB | us |", "|---|---|---|---|---|"]
        for d in att:
            t.append(f"| {d['q']} | {d['g']} | {2 * d['m'] * d['n'] / d['bytes_alg']:.2f}x | "
                     f"{d['bytes_alg'] / 1e6:.1f} | {d['us']} |")
    t += ["", "## batched fc1 (b = 2..32): the shared-memory lookup roof binds from b = 2 (P:L529-530)", "",
          "| b | us | HBM roof us | LDS roof us | % of binding roof | context: dense fp16 cuBLAS us |",
          "|---|---|---|---|---|---|"]
    for d in [x for x in sw if x["b"] == 1 and x["case"] == "fc1"] + [x for x in sw if x["b"] > 1]:
        dn = dense.get(d["b"], {}).get("us", "")
        t.append(f"| {d['b']} | {d['us']} | {d['hbm_roof_us']} | {d['lds_roof_us']} | "
                 f"{100 * d['frac_of_binding_roof']:.1f} | {dn} |")
    if dense:
        t += ["", "Dense fp16 (cuBLAS through torch.matmul, 1.21 GB weight, rotating copies) is a comparison system, "
              "context only (SURVEY K2): it shows where the LUT method's shared-memory roof (P:L529-530) makes a "
              "dense fp16 product faster."]
    if quant:
        t += ["", "## Quantizers (offline step before the path, NEXT-4): dense fp16 fc1 49152 x 12288 -> pack sources", "",
              "| quantizer | q | g | ms | fp16 input GB/s |", "|---|---|---|---|---|"]
        for d in quant:
            t.append(f"| {d['case'][9:]} | {d['q']} | {d['g']} | {d['ms']} | {d['GBps_fp16_in']} |")
    t += ["", "## 96-layer OPT-175B decoder linear stack (tools/stack.py), one token, 1 GPU", "",
          f"{stack['ms_per_token']} ms per token ({stack['GBps_per_gpu']} GB/s over "
          f"{stack['weight_bytes_per_gpu'] / 1e9:.1f} GB of packed weights); per linear (eager): "
          f"{stack['per_linear_us_eager']}.", f"Paper context: {stack['paper_context_ms']}.", ""]
    chk = os.path.join(PROF, f"r{rnd}_stack_tp1_check.json")
    if os.path.exists(p("stack_check.json")):
        d = json.loads(open(p("stack_check.json")).read().strip().splitlines()[-1])
        json.dump(d, open(chk, "w"), indent=1)
    if os.path.exists(chk):
        d = json.load(open(chk))
        v = list(d["parity_rel_l2_sampled"].values())
        t += [f"With `--check` (`r{rnd}_stack_tp1_check.json`): {d['ms_per_token']:.2f} ms per token on that box; "
              f"64 sampled rows of every linear of layers 0 and {d['layers'] - 1} against the fp64 oracle: rel-L2 "
              f"{min(v):.1e} .. {max(v):.1e} (bound 2e-3).", ""]
    open(os.path.join(PROF, f"r{rnd}_sweep.md"), "w").write("\n".join(t) + "\n")
    # sanitizers (tools/sanitize.sh), if that run is present
    san = {t: os.path.join(OUT, f"sanitize_{t}.txt") for t in ("memcheck", "racecheck", "synccheck", "initcheck")}
    closed = any("closed on this pool" in open(v).read() for v in san.values() if os.path.exists(v))
    if all(os.path.exists(v) for v in san.values()) and not closed:
        sl = [f"# Round {int(rnd)} -- compute-sanitizer over every kernel path (SURVEY 4, tier T4)", "",
              "Command: `bash tools/sanitize.sh` (runs `tools/sanitize_case.py` under each tool: GEMV fused and "
              "non-fused with one and many reducers, n and m tails, batched V=2 and V=4, q up to 6, fp32 output, "
              "compact uniform format, the RTN / greedy / alternating quantizers, the fused P2P all-gather at world 1; "
              "every result is checked against "
              "the oracle).", "", "| tool | result | oracle checks passed |", "|---|---|---|"]
        for t, f in san.items():
            txt = open(f).read()
            summ = [l.replace("========= ", "") for l in txt.splitlines() if "SUMMARY" in l]
            sl.append(f"| {t} | {summ[-1] if summ else '?'} | {txt.count(chr(10) + 'ok ') + txt.startswith('ok ')} |")
        sl += ["", "History: the first initcheck run found reads of uninitialised bytes -- warps without any row quad "
               "in a non-fused segment still issued their clamped ring loads at a quad past the range. Fixed (such "
               "warps load nothing); all four tools are clean since."]
        open(os.path.join(PROF, f"r{rnd}_sanitizers.md"), "w").write("\n".join(sl) + "\n")
    print("profiles written for", tag)


if __name__ == "__main__":
    main(*sys.argv[1:])
