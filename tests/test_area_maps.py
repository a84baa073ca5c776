"""The library's FLOP selector (C ABI, runlora_select BY_FLOPS) reproduces the oracle's
Table-1 argmin over the paper's area-map grids (Fig. 2: embedding x rank for
square and 4x-expanding layers at the captions' (b, s); Fig. 3: batch x
sequence length for LlamaMLP 4096->11008, r = 128), including the Eq. 5 region flag and
the closed-form Fig. 3 boundaries (F1 below n = io/(i+o) ≈ 2985, B1 up to n = o = 11008).
"""
import oracle as O

import tools.area_maps as M


def test_fig2_maps_match_oracle():
    for _, mult, b, s in M.FIG2:
        for (e, r), (f, bw, eq5) in M.fig2_grid(mult, b, s).items():
            assert (f, bw) == O.select_by_flops(b * s, e, mult * e, r), (mult, b, s, e, r)
            assert eq5 == O.param_reduction(e, mult * e, r)


def test_fig3_map_matches_oracle_and_closed_form():
    for (b, s), (f, bw) in M.fig3_grid().items():
        n = b * s
        assert (f, bw) == O.select_by_flops(n, 4096, 11008, 128)
        assert f == (1 if n <= 2985 else 2)
        assert bw == (1 if n <= 11008 else 5)
