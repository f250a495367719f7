"""Pins for the oracle's Eq. 4 homomorphic matmul and cost model (no GPU)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import homomm, quant

W = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _q_rows(A, Pi, bits, meta, rnd="rn", u=None):
    """Quantize rows of A [M,Z] in partitions of Pi along Z -> codes, m/s/sums [M, nb]."""
    M, Z = A.shape
    x = A.astype(np.float32).reshape(M, Z // Pi, Pi)
    uu = None if u is None else u.reshape(x.shape)
    c, m, s, sm = quant.quantize(x, bits, meta, rnd, uu)
    return c.reshape(M, Z), m, s, sm


def _q_cols(B, Pi, bits, meta, rnd="rn", u=None):
    c, m, s, sm = _q_rows(B.T, Pi, bits, meta, rnd, None if u is None else u.T)
    return c.T, m.T, s.T, sm.T


def test_w1_real_meta():
    ex = W["eq4"][0]
    A = np.array(ex["A"], np.float64); B = np.array(ex["B"], np.float64)
    ac, am, as_, asum = _q_rows(A, 2, 2, "fp32")
    bc, bm, bs, bsum = _q_cols(B, 2, 2, "fp32")
    assert ac.tolist() == ex["a_codes"] and bc.tolist() == ex["b_codes"]
    # with the exact real scale 2/3 Eq. 4 gives 44
    C = homomm.homomorphic_matmul(ac, am, np.full_like(as_, 2 / 3, dtype=np.float64),
                                  bc, bm, np.full_like(bs, 2 / 3, dtype=np.float64), 2)
    assert abs(C[0, 0] - ex["real_meta_result"]) < 1e-12
    # term by term: 4 + 12 + 4 + 24
    s = 2 / 3
    assert abs(s * s * 9 - 4) < 1e-12 and abs(6 * s * 3 - 12) < 1e-12 and abs(2 * s * 3 - 4) < 1e-12


def test_w2_fp16_meta_and_identity():
    ex = W["eq4"][1]
    A = np.array(ex["A"], np.float64); B = np.array(ex["B"], np.float64)
    ac, am, as_, _ = _q_rows(A, 2, 2, "fp16")
    bc, bm, bs, _ = _q_cols(B, 2, 2, "fp16")
    C = homomm.homomorphic_matmul(ac, am, as_, bc, bm, bs, 2)
    C2 = homomm.dequant_matmul(ac, am, as_, bc, bm, bs, 2)
    assert abs(C[0, 0] - ex["fp16_meta_result"]) < 1e-12
    assert abs(C2[0, 0] - ex["fp16_meta_result"]) < 1e-12


def test_zero_a_gives_zero():
    g = np.random.default_rng(0)
    A = np.zeros((5, 128)); B = g.standard_normal((128, 7))
    ac, am, as_, _ = _q_rows(A, 64, 8, "fp32")
    bc, bm, bs, _ = _q_cols(B, 64, 2, "fp16")
    assert np.all(homomm.homomorphic_matmul(ac, am, as_, bc, bm, bs, 64) == 0)


@pytest.mark.parametrize("Pi,bits", list(itertools.product([32, 64, 128], [2, 4, 8])))
def test_identity_vs_dequantize_then_multiply(Pi, bits):
    # Eq. 4 is algebraically exact: homomorphic == dequantize-then-multiply
    g = np.random.default_rng(Pi * 10 + bits)
    for trial in range(4):
        M, N = g.integers(1, 40, size=2)
        Z = Pi * int(g.integers(1, 4))
        A = (g.standard_normal((M, Z)) * g.uniform(0.1, 5)).astype(np.float16).astype(np.float32)
        B = (g.standard_normal((Z, N)) + g.uniform(-2, 2)).astype(np.float16).astype(np.float32)
        ac, am, as_, asum = _q_rows(A, Pi, 8, "fp32", "sr", g.random(A.shape, dtype=np.float32))
        bc, bm, bs, bsum = _q_cols(B, Pi, bits, "fp16", "sr", g.random(B.shape, dtype=np.float32))
        C = homomm.homomorphic_matmul(ac, am, as_, bc, bm, bs, Pi, asum, bsum)
        C2 = homomm.dequant_matmul(ac, am, as_, bc, bm, bs, Pi)
        scale = np.abs(C2).max() + 1e-30
        assert np.max(np.abs(C - C2)) <= 1e-12 * scale * Z


def test_block_additivity_and_exact_integer_part():
    # per-block integer partials sum to the full integer product a'b'
    g = np.random.default_rng(11)
    a = g.integers(0, 256, size=(17, 192)).astype(np.uint8)
    b = g.integers(0, 4, size=(192, 9)).astype(np.uint8)
    D = homomm.int_blocks(a, b, 64)
    full = np.einsum("iz,zj->ij", a.astype(object), b.astype(object))   # python ints
    assert (D.sum(0).astype(object) == full).all()
    # one block by brute force
    i, j = 3, 5
    assert D[1, i, j] == sum(int(a[i, z]) * int(b[z, j]) for z in range(64, 128))


def test_cached_sums_are_transparent():
    # S:159 sum-cache transparency: passing the stored sums changes nothing
    g = np.random.default_rng(12)
    A = g.standard_normal((8, 128)); B = g.standard_normal((128, 16))
    ac, am, as_, asum = _q_rows(A, 64, 8, "fp32")
    bc, bm, bs, bsum = _q_cols(B, 64, 2, "fp16")
    C1 = homomm.homomorphic_matmul(ac, am, as_, bc, bm, bs, 64)
    C2 = homomm.homomorphic_matmul(ac, am, as_, bc, bm, bs, 64, asum, bsum)
    assert np.array_equal(C1, C2)


def test_sr_eq4_unbiased_brute_force():
    """Exhaustive enumeration (SURVEY c-5 'SR + Eq. 4 unbiased'): A 1x4, B 4x1
    whose scaled values y are multiples of 1/4, so P(round up) = frac(y) is
    exactly the mass of u in {0, 1/4, 1/2, 3/4}.  E[C_hat] over all 4^8
    outcomes equals AB exactly (independent unbiased SR)."""
    A = np.array([[0.0, 0.75, 1.5, 3.0]])          # m=0, s=1 -> y = x
    B = np.array([[1.0], [1.25], [2.5], [4.0]])    # m=1, s=1 -> y = x-1
    levels = np.array([0.0, 0.25, 0.5, 0.75], np.float32)
    total = 0.0
    count = 0
    for ua in itertools.product(levels, repeat=4):
        ac, am, as_, _ = _q_rows(A.astype(np.float32), 4, 2, "fp32", "sr", np.array([ua], np.float32))
        for ub in itertools.product(levels, repeat=4):
            bc, bm, bs, _ = _q_cols(B.astype(np.float32), 4, 2, "fp32", "sr",
                                    np.array(ub, np.float32)[:, None])
            total += homomm.homomorphic_matmul(ac, am, as_, bc, bm, bs, 4)[0, 0]
            count += 1
    assert count == 4 ** 8
    assert abs(total / count - (A @ B)[0, 0]) < 1e-12


@pytest.mark.parametrize("ex", W["cost_model"])
def test_cost_model_examples(ex):
    assert homomm.approximation_cost(ex["M"], ex["N"], ex["Z"], ex["cached"]) == ex["ops"]


def test_decode_cost_closed_form():
    ex = W["decode_cost"]
    d, L = ex["d"], ex["L"]
    assert homomm.decode_approximation_cost(d, L, True) == ex["approx_cached"] == 10 * (d + L)
    assert homomm.dequantization_cost(d, L) == ex["dequant"]
    # uncached = 10(d+L) + 2dL ; P:684 saving vs dequant = 2dL - 10(d+L)
    assert homomm.decode_approximation_cost(d, L, False) == 10 * (d + L) + 2 * d * L
    assert homomm.dequantization_cost(d, L) - homomm.decode_approximation_cost(d, L, False) == \
        2 * d * L - 10 * (d + L)
    assert homomm.quantized_mac_cost(3, 5, 7) == 210
