"""Copies the round-2 profiling run (tools/_r02.sh outputs under gpurun_out/p2/) into
profiles/r02/ and profiles/ncu_summary.json (the traffic figure bench.py reports).

    python tools/refresh_profiles_r02.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_summary as N  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "p2")
PR = os.path.join(ROOT, "profiles", "r02")
ROLES = ["W'ᵀ = (W+AB)ᵀ (identity-tail GEMM, TMA-store epilogue)",
         "Y = X·W'  (main GEMM: 512-wide pair tiles for the leading rows, 256-wide below; TMA-store epilogue)",
         "Z1 = dY·Bᵀ, Z2 = X·A (K-split bf16 blocks, dual; idle warps write A repeated per block)",
         "dA = Xᵀ·Z1, dBᵀ = dYᵀ·Z2 (folded blocks, token-split fp32 slabs)",
         "dX = [dY | Z1 blocks]·[Wᵀ ; Aᵀ ..] (main GEMM; idle warps reduce the dA, dB slabs)"]


def main():
    os.makedirs(PR, exist_ok=True)
    line = [l for l in open(os.path.join(SRC, "bench.log")) if l.startswith("{")][-1]
    open(os.path.join(PR, "bench_line.json"), "w").write(line)
    for src, dst in (("sweep1.jsonl", "sweep_1gpu.jsonl"), ("sweep8.jsonl", "sweep_c4_per_rank_P8.jsonl"),
                     ("gemm.jsonl", "gemm_vs_cublas.jsonl")):
        open(os.path.join(PR, dst), "w").write("".join(l for l in open(os.path.join(SRC, src)) if l.startswith("{")))
    with open(os.path.join(PR, "wq_bench.jsonl"), "w") as f:
        for src in ("wq25.log", "wq21.log"):
            f.write("".join(l for l in open(os.path.join(SRC, src)) if l.startswith("{")))
    full = N.read_rep(os.path.join(SRC, "full.ncu-rep"))
    assert len(full) == len(ROLES), len(full)
    for l, r in zip(full, ROLES):
        l["role"] = r
    json.dump({"source": "ncu --set full --clock-control none, tools/prof_step.py --plan 2,1 --steps 2 "
                         "(the 5 launches of step 2), C2 r=16", "launches": full},
              open(os.path.join(PR, "ncu_full_summary.json"), "w"), indent=1, ensure_ascii=False)
    mains = [full[1], full[4]]
    json.dump({"gemm_main": {"dram_bytes_per_launch": sum(l["dram_read_bytes"] + l["dram_write_bytes"]
                                                         for l in mains) / 2,
                             "source": "profiles/r02/ncu_full_summary.json (ncu --set full, tools/prof_step.py "
                                       "--plan 2,1, mean of the Y and dX GEMMs of step 2)",
                             "launches": mains}},
              open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1, ensure_ascii=False)
    launches = N.read_launches(os.path.join(SRC, "launches.csv"))
    json.dump({"command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                          "--clock-control none --kernel-name-base demangled -k regex:runlora -s 1656 -c 400 "
                          "python bench.py --steps 20 --warmup 5",
               "note": "the library's launches after the 1656 of time-mode selection: warm-up, timed and profile "
                       "steps of C2 r=16 F2+B1 (5 launches per step); cold-cache, serialised (compare shares, "
                       "not absolutes)",
               "launches": launches},
              open(os.path.join(PR, "launches_bench.json"), "w"), indent=1)
    # per-kernel share of a step in the launch list
    per = {}
    for l in launches[:100]:
        per.setdefault(l["kernel"][:40], []).append(l.get("duration_us", 0.0))
    tot = sum(sum(v) for v in per.values())
    print(json.dumps({k: {"launches": len(v), "us": round(sum(v) / 20, 1), "share": round(sum(v) / tot, 3)}
                      for k, v in per.items()}, indent=1))


if __name__ == "__main__":
    main()
