"""GPU parity: quantize_pack (a1-a3) vs the oracle -- codes, packing, fp16/fp32
meta and sums bit-exact for a fixed seed (north star)."""
import numpy as np
import pytest
import torch

import hack_inputs
from oracle import attention as att
from oracle import quant

from .gpu_util import gpu_cfg, hk

pytestmark = pytest.mark.gpu

CASES = [(Pi, b, rnd, dist) for Pi in (32, 64, 128) for b in (2, 4) for rnd in ("sr", "rn")
         for dist in ("normal", "outlier")] + [(64, 2, "sr", "constant"), (64, 2, "sr", "grid"),
                                               (64, 4, "rn", "grid")]


@pytest.mark.parametrize("Pi,bits,rnd,dist", CASES)
def test_quantize_k_bit_exact(Pi, bits, rnd, dist):
    h = hk()
    rows, H, pos0 = 77, 3, 1234
    ocfg = att.Config(Hq=H, Hkv=H, Pi=Pi, bits=bits, kv_round=rnd, q_round=rnd, seed=0xABCDEF12345, layer=7,
                      head_base=2)
    g = hack_inputs.rng(1, Pi, bits)
    x = hack_inputs.tensor(g, (rows, H, 128), dist, grid_bits=bits, partition=Pi)
    codes, m, s, sm = att.quantize_k(ocfg, x, np.arange(pos0, pos0 + rows), rng_id=99)
    cfg = gpu_cfg(ocfg)
    nb = 128 // Pi
    sb = 1 if bits + int(np.log2(Pi)) <= 8 else 2
    xc = torch.from_numpy(x).cuda()
    gc = torch.zeros((rows, H, 128 * bits // 8), dtype=torch.uint8, device="cuda")
    gm = torch.zeros((rows, H, nb, 2), dtype=torch.float16, device="cuda")
    gs = torch.zeros((rows, H, nb), dtype=torch.uint8 if sb == 1 else torch.int16, device="cuda")
    h.quantize_pack(cfg, h.QMODE_K, xc, gc, gm, gs, pos0=pos0, head0=ocfg.head_base, rng_id=99)
    torch.cuda.synchronize()
    assert np.array_equal(gc.cpu().numpy(), quant.pack(codes, bits))
    gmn = gm.cpu().numpy()
    assert np.array_equal(gmn[..., 0].astype(np.float32), m) and np.array_equal(gmn[..., 1].astype(np.float32), s)
    gsn = gs.cpu().numpy().astype(np.int64) & (0xFF if sb == 1 else 0xFFFF)
    assert np.array_equal(gsn, sm)


@pytest.mark.parametrize("Pi,bits,rnd", [(32, 2, "sr"), (64, 2, "sr"), (128, 2, "sr"), (64, 4, "sr"),
                                         (64, 2, "rn"), (128, 4, "rn")])
def test_quantize_v_bit_exact(Pi, bits, rnd):
    h = hk()
    nblk, H = 3, 2
    pos0 = 5 * Pi
    ocfg = att.Config(Hq=H, Hkv=H, Pi=Pi, bits=bits, kv_round=rnd, seed=77, layer=3, head_base=1)
    g = hack_inputs.rng(2, Pi, bits)
    x = hack_inputs.tensor(g, (nblk * Pi, H, 128), "outlier")
    cfg = gpu_cfg(ocfg)
    sb = 1 if bits + int(np.log2(Pi)) <= 8 else 2
    gc = torch.zeros((nblk, H, 128, Pi * bits // 8), dtype=torch.uint8, device="cuda")
    gm = torch.zeros((nblk, H, 128, 2), dtype=torch.float16, device="cuda")
    gs = torch.zeros((nblk, H, 128), dtype=torch.uint8 if sb == 1 else torch.int16, device="cuda")
    h.quantize_pack(cfg, h.QMODE_V, torch.from_numpy(x).cuda(), gc, gm, gs, pos0=pos0, head0=1, rng_id=5)
    torch.cuda.synchronize()
    for j in range(nblk):
        c, m, s, sm = att.quantize_v_block(ocfg, x[j * Pi:(j + 1) * Pi], pos0 + j * Pi, rng_id=5)
        assert np.array_equal(gc[j].cpu().numpy(), quant.pack(c, bits))
        gmn = gm[j].cpu().numpy()
        assert np.array_equal(gmn[..., 0].astype(np.float32), m) and np.array_equal(gmn[..., 1].astype(np.float32), s)
        assert np.array_equal(gs[j].cpu().numpy().astype(np.int64) & (0xFF if sb == 1 else 0xFFFF), sm)


@pytest.mark.parametrize("Pi,rnd", [(32, "sr"), (64, "sr"), (128, "sr"), (64, "rn")])
def test_quantize_q_bit_exact(Pi, rnd):
    h = hk()
    rows, Hq, Hkv = 50, 8, 2
    ocfg = att.Config(Hq=Hq, Hkv=Hkv, Pi=Pi, q_round=rnd, seed=3, head_base=1)
    q = hack_inputs.tensor(hack_inputs.rng(3, Pi), (rows, Hq, 128), "normal")
    codes, m, s, sm = att.quantize_q(ocfg, q, np.arange(10, 10 + rows), rng_id=4)
    cfg = gpu_cfg(ocfg)
    nb = 128 // Pi
    gc = torch.zeros((rows, Hq, 128), dtype=torch.uint8, device="cuda")
    gm = torch.zeros((rows, Hq, nb, 2), dtype=torch.float32, device="cuda")
    gs = torch.zeros((rows, Hq, nb), dtype=torch.int16, device="cuda")
    h.quantize_pack(cfg, h.QMODE_Q, torch.from_numpy(q).cuda(), gc, gm, gs, pos0=10,
                    head0=ocfg.head_base * ocfg.G, rng_id=4)
    torch.cuda.synchronize()
    assert np.array_equal(gc.cpu().numpy(), codes)
    gmn = gm.cpu().numpy()
    assert np.array_equal(gmn[..., 0], m) and np.array_equal(gmn[..., 1], s)
    assert np.array_equal(gs.cpu().numpy().astype(np.int64) & 0xFFFF, sm)
