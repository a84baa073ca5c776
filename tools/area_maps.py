"""Areas of the best forward/backward variant (Fig. 2, and Fig. 3,
P:255-275) regenerated from the library's selector.

    python tools/area_maps.py [--out profiles/r01/area_maps] [--measured]

FLOP criterion (no GPU needed): Table 1 argmin per cell.
  fig2_<square|expand>_b<b>_s<s>.csv   rows: embedding e, columns: rank r; cell "F?+B?" and
                                        "*" where Eq. 5 holds (the paper's dashed-line region)
  fig3_llama_mlp_r128_<fwd|bwd>.csv     rows: batch b, columns: sequence length s
--measured adds fig3_llama_mlp_r128_time.csv: the time criterion on this GPU over a coarse
(b, s) grid (each cell: time pick, FLOP pick, candidate medians in µs).
"""
import argparse
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_03415_b200 import runlora as rl  # noqa: E402

FIG2 = [("square", 1, 2, 100), ("expand", 4, 2, 100), ("square", 1, 20, 1024), ("expand", 4, 1, 600)]
EMB = [256, 512, 768, 1024, 1536, 2048, 3072, 4096, 5120, 6144, 8192]
RANKS = [8, 16, 32, 64, 128, 256, 512, 1024]
BATCH = [1, 2, 4, 8, 16, 32, 64]
SEQ = [128, 256, 512, 1024, 2048, 4096]


def flop_pick(n, k, m, r):
    p = rl.select_by_flops(rl.make_shape(n, k, m, r, rl.BF16))
    return int(p.fwd), int(p.bwd)


def fig2_grid(mult, b, s):
    """{(e, r): (fwd, bwd, eq5)} over embedding e and rank r <= e (i = e, o = mult*e)."""
    out = {}
    for e in EMB:
        for r in RANKS:
            if r <= e:
                f, bw = flop_pick(b * s, e, mult * e, r)
                out[(e, r)] = (f, bw, r * (e + mult * e) < e * mult * e)
    return out


def fig3_grid(k=4096, m=11008, r=128):
    return {(b, s): flop_pick(b * s, k, m, r) for b in BATCH for s in SEQ}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r01/area_maps")
    ap.add_argument("--measured", action="store_true")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    for name, mult, b, s in FIG2:
        g = fig2_grid(mult, b, s)
        with open(os.path.join(a.out, f"fig2_{name}_b{b}_s{s}.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["e \\ r"] + RANKS)
            for e in EMB:
                w.writerow([e] + [f"F{g[(e, r)][0]}+B{g[(e, r)][1]}{'*' if g[(e, r)][2] else ''}" if (e, r) in g else ""
                                  for r in RANKS])
    g3 = fig3_grid()
    for idx, tag in ((0, "fwd"), (1, "bwd")):
        with open(os.path.join(a.out, f"fig3_llama_mlp_r128_{tag}.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["b \\ s"] + SEQ)
            for b in BATCH:
                w.writerow([b] + [f"{'F' if idx == 0 else 'B'}{g3[(b, s)][idx]}" for s in SEQ])
    if a.measured:
        import torch
        h = rl.handle(0)
        k, m, r = 4096, 11008, 128
        W = torch.randn(k, m, device="cuda").mul_(k ** -0.5).to(torch.bfloat16)
        A = torch.randn(k, r, device="cuda").mul_(k ** -0.5).to(torch.bfloat16)
        B = torch.randn(r, m, device="cuda").mul_(r ** -0.5).to(torch.bfloat16)
        rows = []
        for b in (1, 4, 16, 64):
            for s in (128, 512, 2048):
                n = b * s
                ops = {"X": torch.randn(n, k, device="cuda").to(torch.bfloat16), "W": W, "A": A, "B": B,
                       "dY": torch.randn(n, m, device="cuda").to(torch.bfloat16),
                       "Y": torch.empty(n, m, device="cuda", dtype=torch.bfloat16),
                       "dX": torch.empty(n, k, device="cuda", dtype=torch.bfloat16),
                       "dA": torch.empty(k, r, device="cuda"), "dB": torch.empty(r, m, device="cuda")}
                p = h.select(rl.make_shape(n, k, m, r, rl.BF16), rl.BY_TIME, ops=ops, grad_dtype=rl.F32)
                d = p.as_dict()
                rows.append([b, s, n, f"F{p.fwd}+B{p.bwd}", f"F{p.flops_fwd_pick}+B{p.flops_bwd_pick}",
                             json.dumps({**{f"F{v}": round(t, 1) for v, t in d["time_fwd_us"].items()},
                                         **{f"B{v}": round(t, 1) for v, t in d["time_bwd_us"].items()}})])
                del ops
                torch.cuda.empty_cache()
        with open(os.path.join(a.out, "fig3_llama_mlp_r128_time.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["b", "s", "n", "time_pick", "flops_pick", "candidates_us"])
            w.writerows(rows)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
