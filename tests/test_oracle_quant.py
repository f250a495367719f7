"""Pins for the oracle's RNG, quantizer and packer (no GPU).

Each test pins the oracle against something other than itself: known-answer
vectors, the paper/SPEC worked examples (tests/golden), closed forms,
statistical laws, exhaustive enumeration."""
import json
import os

import numpy as np
import pytest

from oracle import philox, quant

GOLD = os.path.join(os.path.dirname(__file__), "golden")
W = json.load(open(os.path.join(GOLD, "worked_examples.json")))
KAT = json.load(open(os.path.join(GOLD, "philox_kat.json")))


@pytest.mark.parametrize("vec", KAT["vectors"])
def test_philox_kat(vec):
    c = [int(x, 16) for x in vec["ctr"]]
    k = [int(x, 16) for x in vec["key"]]
    out = philox.philox4x32_10(*c, *k)
    assert [int(o) for o in out] == [int(x, 16) for x in vec["out"]]


def test_counter_map_is_injective_and_in_range():
    # K stream: every (t, c) hits a distinct (n, w); V stream likewise.
    d = 128
    t = np.arange(300)
    for fn in ("rowwise", "colwise"):
        if fn == "rowwise":
            n = (t[:, None] * d + np.arange(d)[None, :]) >> 2
            w = np.arange(d)[None, :] & 3
        else:
            n = (t[:, None] >> 2) * d + np.arange(d)[None, :]
            w = t[:, None] & 3
        key = (n * 4 + w).ravel()
        assert len(np.unique(key)) == key.size
    u = philox.uniforms_rowwise(1, 2, 3, philox.TAG_K, 4, np.arange(64), d)
    assert u.dtype == np.float32 and (u >= 0).all() and (u < 1).all()
    # 24-bit resolution: u * 2^24 is an integer
    assert np.all(np.floor(u.astype(np.float64) * 2 ** 24) == u.astype(np.float64) * 2 ** 24)


def test_uniforms_are_uniform():
    u = philox.uniforms_rowwise(7, 0, 0, philox.TAG_Q, 0, np.arange(2000), 128).ravel()
    # mean 1/2, var 1/12 within 5 sigma
    n = u.size
    assert abs(u.mean() - 0.5) < 5 * np.sqrt(1 / 12 / n)
    hist, _ = np.histogram(u, bins=16, range=(0, 1))
    exp = n / 16
    chi2 = ((hist - exp) ** 2 / exp).sum()
    assert chi2 < 50  # 15 dof; p ~ 1e-5


@pytest.mark.parametrize("ex", W["partition_stats"])
def test_partition_stats_spec(ex):
    m, s = quant.partition_stats(np.array(ex["x"], np.float32), ex["bits"], meta="fp32")
    assert float(m) == ex["m"]
    assert abs(float(s) - ex["s"]) < 1e-7


@pytest.mark.parametrize("ex", W["quantize_fp16_meta_rn"])
def test_quantize_worked_examples(ex):
    x = np.array(ex["x"], np.float16).astype(np.float32)
    c, m, s, sm = quant.quantize(x, ex["bits"], "fp16", "rn")
    assert c.tolist() == ex["codes"]
    assert float(m) == ex["m"] and float(s) == ex["s"] and int(sm) == ex["sum"]
    if "dequant" in ex:
        assert quant.dequantize(c, m, s).tolist() == ex["dequant"]


def test_constant_partition_scale_zero():
    # constant -> all codes 0, dequantize returns the constant (reading R5)
    x = np.full((3, 64), 1.7001953125, np.float32)
    for rnd, u in (("rn", None), ("sr", np.random.default_rng(0).random((3, 64), dtype=np.float32))):
        c, m, s, sm = quant.quantize(x, 2, "fp16", rnd, u)
        assert (c == 0).all() and (s == 0).all() and (sm == 0).all()
        assert np.all(quant.dequantize(c, m, s) == x)


def test_reconstruction_error_bounds():
    # RN |x_hat - x| <= s/2 ; SR < s  (s = stored scale); random 8x64, b in {2,4,8}
    g = np.random.default_rng(1)
    x = g.standard_normal((8, 64)).astype(np.float16).astype(np.float32)
    u = g.random((8, 64), dtype=np.float32)
    for b in (2, 4, 8):
        for rnd in ("rn", "sr"):
            c, m, s, _ = quant.quantize(x, b, "fp32", rnd, u)
            err = np.abs(quant.dequantize(c, m, s) - x)
            bound = (0.5 if rnd == "rn" else 1.0) * s[:, None].astype(np.float64)
            assert np.all(err <= bound * (1 + 1e-5) + 1e-7)
            assert c.max() <= (1 << b) - 1


def test_fp16_meta_codes_never_exceed_range():
    # R4: codes are computed against the rounded fp16 scale; clamp keeps them in range
    g = np.random.default_rng(2)
    x = (g.standard_normal((4000, 64)) * 3).astype(np.float16).astype(np.float32)
    c, m, s, _ = quant.quantize(x, 2, "fp16", "rn")
    assert c.max() == 3 and c.min() == 0
    # the max element quantizes to 2^b-1 or (if s16 rounded up) to 2^b-1 after RN
    hi = x.argmax(-1)
    assert np.all(c[np.arange(4000), hi] == 3)


def test_sr_integer_is_deterministic_and_half_is_fair():
    # 2.0 -> 2 with probability 1; 1.5 -> 1 or 2 with p = 1/2
    n = 100000
    g = np.random.default_rng(3)
    # partition [0, 2, 3] with s = 1 -> y = [0, 2, 3]: integer, deterministic
    x = np.tile(np.array([0, 2, 3], np.float32), (n, 1))
    u = g.random(x.shape, dtype=np.float32)
    c, _, _, _ = quant.quantize(x, 2, "fp32", "sr", u)
    assert (c == np.array([0, 2, 3])).all()
    # partition [0, 1.5, 3] -> y = 1.5
    x = np.tile(np.array([0, 1.5, 3], np.float32), (n, 1))
    c, _, _, _ = quant.quantize(x, 2, "fp32", "sr", g.random(x.shape, dtype=np.float32))
    p = (c[:, 1] == 2).mean()
    assert abs(p - 0.5) < 4 * np.sqrt(0.25 / n)
    assert set(np.unique(c[:, 1])) == {1, 2}


@pytest.mark.parametrize("target", [0.25, 0.1, 0.5, 0.9, 2.75])
def test_sr_unbiased_with_philox(target):
    # S:58 / S:593: empirical mean over 1e5 Philox counters within 4 sigma.
    # Partition [0, target, 3] (s = 1, m = 0), u from the real counter map.
    n = 100000
    x = np.tile(np.array([0, target, 3], np.float32), (n, 1))
    u = philox.uniforms(99, 0, 0, philox.TAG_K, 0, np.arange(n), np.zeros(n, np.int64))
    uu = np.zeros(x.shape, np.float32)
    uu[:, 1] = u
    c, m, s, _ = quant.quantize(x, 2, "fp32", "sr", uu)
    xhat = quant.dequantize(c, m, s)[:, 1]
    f = target - np.floor(target)
    sigma = np.sqrt(f * (1 - f) / n)
    assert abs(xhat.mean() - target) <= 4 * sigma + 1e-9


@pytest.mark.parametrize("ex", W["pack"])
def test_pack_examples(ex):
    assert quant.pack(np.array(ex["codes"]), ex["bits"]).tolist() == ex["bytes"]


@pytest.mark.parametrize("bits", [2, 4, 8])
def test_pack_round_trip(bits):
    g = np.random.default_rng(4)
    codes = g.integers(0, 1 << bits, size=(10000,)).astype(np.uint8)
    p = quant.pack(codes, bits)
    assert p.size == 10000 * bits // 8
    assert (quant.unpack(p, bits, 10000) == codes).all()
    # LSB-first: code j of byte i sits at bits [j*b, (j+1)*b)
    if bits < 8:
        per = 8 // bits
        j = 5
        assert (p[j // per] >> ((j % per) * bits)) & ((1 << bits) - 1) == codes[j]


@pytest.mark.parametrize("ex", W["sum_width"])
def test_sum_width(ex):
    assert quant.sum_width_bits(ex["bits"], ex["partition"]) == ex["width"]


def test_sum_all_threes():
    # a Pi=64, b=2 sum needs at most 8 bits (upper bound 64*3 = 192).
    ex = W["all_codes_3_sum"]
    assert ex["partition"] * 3 == ex["sum"] < 2 ** quant.sum_width_bits(2, ex["partition"])
    # the quantizer's sums are exact code sums and never exceed the bound
    g = np.random.default_rng(6)
    x = np.concatenate([np.zeros((500, 1)), g.random((500, 63)) * 0.01 + 3.0], 1).astype(np.float32)
    c, _, _, sm = quant.quantize(x, 2, "fp32", "rn")
    assert (sm == c.astype(np.int64).sum(-1)).all() and sm.max() <= 192 and sm.max() >= 150


def test_partition_independence():
    # changing one partition never changes another's codes or meta
    g = np.random.default_rng(5)
    x = g.standard_normal((6, 64)).astype(np.float16).astype(np.float32)
    u = g.random(x.shape, dtype=np.float32)
    c1, m1, s1, _ = quant.quantize(x, 2, "fp16", "sr", u)
    x2 = x.copy()
    x2[3] *= 7
    c2, m2, s2, _ = quant.quantize(x2, 2, "fp16", "sr", u)
    keep = [0, 1, 2, 4, 5]
    assert (c1[keep] == c2[keep]).all() and (m1[keep] == m2[keep]).all() and (s1[keep] == s2[keep]).all()
