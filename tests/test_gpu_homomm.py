"""GPU parity: hack_homomorphic_matmul (N9 test export: tcgen05 kind::i8 MMA core) vs the
oracle.  Per-block int32 partials D_beta bit-exact; C = sum_beta Eq. 4 within 1e-3
relative of the oracle's fp64 Eq. 4 and of dequantize-then-multiply."""
import numpy as np
import pytest
import torch

from oracle import homomm, quant

from .gpu_util import hk

pytestmark = pytest.mark.gpu


def make_operands(g, M, N, Z, Pi, bits):
    A = (g.standard_normal((M, Z)) * g.uniform(0.2, 3)).astype(np.float16).astype(np.float32)
    B = (g.standard_normal((Z, N)) + g.uniform(-1, 1)).astype(np.float16).astype(np.float32)
    ua = g.random((M, Z // Pi, Pi), dtype=np.float32)
    ub = g.random((N, Z // Pi, Pi), dtype=np.float32)
    ac, am, as_, asum = quant.quantize(A.reshape(M, Z // Pi, Pi), 8, "fp32", "sr", ua)
    bc, bm, bs, bsum = quant.quantize(B.T.reshape(N, Z // Pi, Pi), bits, "fp16", "sr", ub)
    return ac.reshape(M, Z), am, as_, asum, bc.reshape(N, Z), bm, bs, bsum


@pytest.mark.parametrize("M,N,Z,Pi,bits", [(128, 64, 128, 64, 2), (200, 100, 256, 64, 2), (77, 33, 128, 32, 2),
                                           (130, 70, 256, 128, 2), (128, 64, 512, 64, 4), (65, 129, 128, 32, 4),
                                           (300, 200, 1024, 64, 2)])
def test_homomorphic_matmul_matches_oracle(M, N, Z, Pi, bits):
    h = hk()
    g = np.random.default_rng(M * 7 + N + Z + bits)
    ac, am, as_, asum, bc, bm, bs, bsum = make_operands(g, M, N, Z, Pi, bits)
    cfg = h.config(partition=Pi, kv_bits=bits)
    sb = 1 if bits + int(np.log2(Pi)) <= 8 else 2
    nb = Z // Pi
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    a_meta = t(np.stack([am, as_], -1).astype(np.float32))
    b_meta = t(np.stack([bm, bs], -1).astype(np.float16))
    b_sums = t(bsum.astype(np.uint8 if sb == 1 else np.uint16).view(np.uint8 if sb == 1 else np.int16))
    dblk = torch.zeros((nb, M, N), dtype=torch.int32, device="cuda")
    c = torch.zeros((M, N), dtype=torch.float32, device="cuda")
    h.homomorphic_matmul(cfg, t(ac), a_meta, t(asum.astype(np.uint16).view(np.int16)), t(quant.pack(bc, bits)),
                         b_meta, b_sums, M, N, Z, c, d_blocks=dblk)
    torch.cuda.synchronize()
    D = homomm.int_blocks(ac, bc.T, Pi)
    assert np.array_equal(dblk.cpu().numpy(), D)
    C_ref = homomm.homomorphic_matmul(ac, am, as_, bc.T, bm.T, bs.T, Pi)
    C_twin = homomm.dequant_matmul(ac, am, as_, bc.T, bm.T, bs.T, Pi)
    cg = c.cpu().numpy()
    scale = np.abs(C_ref).max()
    assert np.abs(cg - C_ref).max() <= 1e-3 * scale
    assert np.abs(cg - C_twin).max() <= 1e-3 * scale
