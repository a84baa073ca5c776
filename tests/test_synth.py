"""The seeded input generators: determinism, chunking, laws, sampling."""
import numpy as np
import torch

import synth


def test_determinism_and_dtype():
    c = synth.C1
    a = synth.draw(c, synth.T_X, (16, 8))
    b = synth.draw(c, synth.T_X, (16, 8))
    assert a.dtype == torch.float32 and torch.equal(a, b)
    c2 = synth.C2[16]
    x = synth.draw(c2, synth.T_W, (8, 8))
    assert x.dtype == torch.bfloat16


def test_chunked_equals_single_draw(monkeypatch):
    c = synth.case("t", 0, 0, 64, 32, 32, 4, "f32")
    whole = synth.draw(c, synth.T_X, (64, 32))
    monkeypatch.setattr(synth, "_CHUNK_ELEMS", 32 * 5)
    chunked = synth.draw(c, synth.T_X, (64, 32))
    assert torch.equal(whole, chunked)


def test_laws():
    c = synth.C2[16]
    assert abs(c.std[synth.T_W] - 1 / 64) < 1e-15
    assert abs(c.std[synth.T_B] - 0.25) < 1e-15
    w = synth.draw(c, synth.T_W, (512, 512)).float()
    assert abs(w.std().item() * 64 - 1) < 0.02


def test_sample_rows():
    rows = synth.sample_rows(8192, P=4, count=512)
    assert rows[0] == 0 and rows[-1] == 8191
    assert len(rows) == 512 and len(np.unique(rows)) == 512
    for b in (2048, 4096, 6144):
        assert b in rows and b - 1 in rows
    assert len(synth.sample_rows(10, count=512)) == 10
