"""Copies one profiling run (tools/_p*.sh outputs under gpurun_out/<prefix>_*) into
profiles/r01/ and refreshes the generated tables of BASELINE.md §4 and profiles/r01/SUMMARY.md.

    python tools/refresh_profiles.py p4
"""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as N  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PR = os.path.join(ROOT, "profiles", "r01")
ROLES = ["W'ᵀ = (W+AB)ᵀ (identity-tail GEMM, TMA-store epilogue)",
         "Y = X·W'  (main GEMM: 512-wide pair tiles for the leading rows, 256-wide below; TMA-store epilogue)",
         "A repeated for the dX tail", "Z1 = dY·Bᵀ, Z2 = X·A (K-split bf16 blocks, dual)",
         "dA = Xᵀ·Z1, dBᵀ = dYᵀ·Z2 (folded blocks, token splits)",
         "dX = [dY | Z1 blocks]·[Wᵀ ; Aᵀ ..] (main GEMM, concat-K tail; 512/256-wide tiles)",
         "fixed-order reducer -> dA, dB fp32"]


def main():
    pre = sys.argv[1]
    g = lambda s: os.path.join(ROOT, "gpurun_out", f"{pre}_{s}")  # noqa: E731
    line = [l for l in open(g("bench.log")) if l.startswith("{")][-1]
    open(os.path.join(PR, "bench_line.json"), "w").write(line)
    for src, dst in (("sweep1.jsonl", "sweep_1gpu.jsonl"), ("sweep8.jsonl", "sweep_c4_per_rank_P8.jsonl"),
                     ("stack.jsonl", "stack_bench.jsonl")):
        open(os.path.join(PR, dst), "w").write(open(g(src)).read())
    full = N.read_rep(g("full.ncu-rep"))
    assert len(full) == len(ROLES), len(full)
    for l, r in zip(full, ROLES):
        l["role"] = r
    json.dump({"source": "ncu --set full --clock-control none, tools/prof_step.py --plan 2,1 --steps 2 "
                         "(launches of step 2), C2 r=16", "launches": full},
              open(os.path.join(PR, "ncu_full_summary.json"), "w"), indent=1, ensure_ascii=False)
    mains = [full[1], full[5]]
    json.dump({"gemm_main": {"dram_bytes_per_launch": sum(l["dram_read_bytes"] + l["dram_write_bytes"]
                                                         for l in mains) / 2,
                             "source": "profiles/r01/ncu_full_summary.json (ncu --set full, tools/prof_step.py "
                                       "--plan 2,1, mean of the Y and dX GEMMs of step 2)",
                             "launches": mains}},
              open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1, ensure_ascii=False)
    json.dump({"command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                          "--clock-control none -c 2000 python bench.py --steps 20 --warmup 3 --no-cpu-baseline",
               "note": "cold-cache, serialised per-launch times (compare shares, not absolutes); includes plan "
                       "selection, the e2e leg and the default-chain comparator (nvjet = cuBLAS)",
               "launches": N.read_launches(g("launches.csv"))},
              open(os.path.join(PR, "launches_bench.json"), "w"), indent=1)
    # BASELINE.md §4 sweep table
    rows = [json.loads(l) for l in open(os.path.join(PR, "sweep_1gpu.jsonl")) if l.startswith("{")]
    rows += [json.loads(l) for l in open(os.path.join(PR, "sweep_c4_per_rank_P8.jsonl")) if l.startswith("{")]
    tab = "\n".join(f"| {r['config']} | {r['n']} | {r['k']}×{r['m']} | {r['r']} | {r['plan_time']} / {r['plan_flops']} "
                    f"| {r['ms_per_step'] * 1e3:.1f} | {r['tokens_per_s'] / 1e6:.2f} M | {r['tflops']:.0f} | "
                    f"{r['ms_default_chain'] * 1e3:.1f} | {r['speedup_vs_default']:.2f}× |" for r in rows)
    p = os.path.join(ROOT, "BASELINE.md")
    s = open(p).read()
    hdr = ("| config | n | k×m | r | plan (time / FLOPs) | µs/step | tokens/s | TFLOP/s | default chain µs | speedup |\n"
           "|---|---|---|---|---|---|---|---|---|---|\n")
    i = s.index(hdr) + len(hdr)
    j = s.index("\n\n", i)
    s = s[:i] + tab + s[j:]
    st = json.loads(open(os.path.join(PR, "stack_bench.jsonl")).read().splitlines()[0])
    s = re.sub(r"\d+ ms/step \([\d.]+ k tokens/s\) vs \d+ ms with every linear as\nthe default chain: [\d.]+×\.",
               f"{st['ms_per_step']:.0f} ms/step ({st['tokens_per_s'] / 1e3:.1f} k tokens/s) vs "
               f"{st['default_chain_ms']:.0f} ms with every linear as\nthe default chain: {st['speedup']:.2f}×.", s)
    open(p, "w").write(s)
    # SUMMARY.md ncu table
    p = os.path.join(PR, "SUMMARY.md")
    s = open(p).read()
    i = s.index("## One forward2 + backward1 step")
    j = s.index("## Findings this round")
    rows = "\n".join(f"| {l['role']} | `{l['kernel'][:38]}` | {l['duration_us']:.1f} | {l['dram_read_bytes'] / 1e6:.1f} / "
                     f"{l['dram_write_bytes'] / 1e6:.1f} | {l['tensor_pipe_pct']:.1f} | {l['dram_throughput_pct']:.1f} |"
                     for l in full)
    tot = sum(l["duration_us"] for l in full)
    s = s[:i] + (f"## One forward2 + backward1 step (ncu, cold cache, serialised; {tot:.0f} µs total)\n\n"
                 "| launch | kernel | µs | DRAM read / write (MB) | tensor pipe % | DRAM % |\n"
                 "|---|---|---|---|---|---|\n" + rows + "\n\n") + s[j:]
    open(p, "w").write(s)
    d = json.loads(line)
    r = d["roofline"]
    print(f"value {d['value'] / 1e6:.2f} M tok/s, {d['ms_per_step'] * 1e3:.1f} us/step, x{d['speedup_vs_default']:.3f} "
          f"(chain {d['default_chain']['ms_per_step'] * 1e3:.1f}), main {r['achieved']:.0f} TF/s frac {r['frac']:.3f} "
          f"burst {r['frac_of_burst']:.3f}, e2e {d['e2e']['value'] / 1e6:.2f} M, clocks {d['clocks']}, "
          f"cpu {d['cpu_baseline']['value'] / 1e3:.1f} k")
    for k, v in r["hbm_kernels"].items():
        print(k, round(v.get("achieved_work", 0)))


if __name__ == "__main__":
    main()
