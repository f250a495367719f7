"""GPU parity: hack_homomorphic_matmul (N9 test export: the prefill kernel's tcgen05 kind::i8
configuration, s8 (a' - 128) x u8 (2 b')) vs the oracle.  Per-block int32 partials D_beta
bit-exact at every Z (no CUDA-core fallback exists); C = sum_beta Eq. 4 per ELEMENT within
1e-5 of sum_beta max|a_hat| sum|b_hat| (a bound of every term the fp32 epilogue adds) and
per row within 1e-3
(R18) of the oracle's fp64 Eq. 4 and of dequantize-then-multiply."""
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
                                           (300, 200, 1024, 64, 2), (129, 65, 2048, 128, 4),
                                           (64, 300, 4096, 32, 2)])
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
    a_hat = np.repeat(as_, Pi, axis=1) * ac + np.repeat(am, Pi, axis=1)          # [M, Z]
    b_hat = np.repeat(bs, Pi, axis=1) * bc + np.repeat(bm, Pi, axis=1)          # [N, Z]
    # per-element scale bounding every Eq. 4 term: sum_beta max_z|a_hat| * sum_z |b_hat| over the block
    amax = np.abs(a_hat).reshape(M, nb, Pi).max(-1)                             # [M, nb]
    bsum = np.abs(b_hat).reshape(N, nb, Pi).sum(-1)                             # [N, nb]
    mag = amax @ bsum.T
    assert (np.abs(cg - C_ref) <= 1e-5 * mag + 1e-30).all()
    for ref in (C_ref, C_twin):
        row = np.abs(cg - ref).max(1) / np.maximum(np.abs(ref).max(1), 1e-6)
        assert row.max() <= 1e-3
