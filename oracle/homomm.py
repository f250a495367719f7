"""Homomorphic matrix multiplication, Eq. 4, block form,
the dequantize-then-multiply twin, and the paper's cost model.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

For C = A B with A [M, Z] partitioned along rows' inner dim and B [Z, N]
partitioned along columns' inner dim (fig:hoq_matmul), per block beta
of Pi inner elements ("A1 B1^T + A2 B2^T"):

  c_ij ~= sum_beta [ s_a s_b sum_z a'_iz b'_zj  +  m_b s_a sum_z a'_iz
                     + m_a s_b sum_z b'_zj        +  Z m_a m_b ]          (Eq. 4)

with Z = Pi inside a block.  The integer part D_beta = sum_z a' b' is exact
(int64 here); every other term is fp64.
"""
from __future__ import annotations

import numpy as np


def int_blocks(a_codes: np.ndarray, b_codes: np.ndarray, partition: int) -> np.ndarray:
    """D[beta, i, j] = sum_{z in beta} a'_iz b'_zj, exact int64.
    a_codes [M, Z], b_codes [Z, N] (uint8)."""
    M, Z = a_codes.shape
    Z2, N = b_codes.shape
    if Z != Z2 or Z % partition:
        raise ValueError("inner dims must agree and be a multiple of Pi")
    nb = Z // partition
    D = np.empty((nb, M, N), dtype=np.int64)
    a = a_codes.astype(np.int64)
    b = b_codes.astype(np.int64)
    for beta in range(nb):
        sl = slice(beta * partition, (beta + 1) * partition)
        D[beta] = a[:, sl] @ b[sl, :]
    return D


def homomorphic_matmul(a_codes, a_m, a_s, b_codes, b_m, b_s, partition,
                       a_sums=None, b_sums=None, return_blocks=False):
    """Eq. 4 per block, summed over blocks.  fp64 result [M, N].

    a_m, a_s, a_sums : [M, nb]   (per row i, block beta)
    b_m, b_s, b_sums : [nb, N]   (per block beta, column j)
    Sums default to the exact code sums (summation elimination, only
    changes *when* they are computed, never their value)."""
    D = int_blocks(a_codes, b_codes, partition)
    nb = D.shape[0]
    M, N = D.shape[1], D.shape[2]
    if a_sums is None:
        a_sums = a_codes.astype(np.int64).reshape(M, nb, partition).sum(-1)
    if b_sums is None:
        b_sums = b_codes.astype(np.int64).reshape(nb, partition, N).sum(1)
    a_m = np.asarray(a_m, np.float64); a_s = np.asarray(a_s, np.float64)
    b_m = np.asarray(b_m, np.float64); b_s = np.asarray(b_s, np.float64)
    C = np.zeros((M, N), dtype=np.float64)
    for beta in range(nb):
        sa, ma, SA = a_s[:, beta][:, None], a_m[:, beta][:, None], a_sums[:, beta][:, None]
        sb, mb, SB = b_s[beta][None, :], b_m[beta][None, :], b_sums[beta][None, :]
        C += (sa * sb * D[beta]          # s_a s_b sum a'b'
              + mb * sa * SA             # m_b s_a sum a'
              + ma * sb * SB             # m_a s_b sum b'
              + partition * ma * mb)     # Z m_a m_b
    return (C, D) if return_blocks else C


def dequant_matmul(a_codes, a_m, a_s, b_codes, b_m, b_s, partition) -> np.ndarray:
    """Twin: dequantize both operands (x_hat = s x' + m), then multiply."""
    M, Z = a_codes.shape
    N = b_codes.shape[1]
    nb = Z // partition
    a_hat = (np.repeat(np.asarray(a_s, np.float64), partition, axis=1) * a_codes +
             np.repeat(np.asarray(a_m, np.float64), partition, axis=1))
    b_hat = (np.repeat(np.asarray(b_s, np.float64), partition, axis=0) * b_codes +
             np.repeat(np.asarray(b_m, np.float64), partition, axis=0))
    assert a_hat.shape == (M, Z) and b_hat.shape == (Z, N) and nb * partition == Z
    return a_hat @ b_hat


# ---- cost model -------------------------------

def approximation_cost(M: int, N: int, Z: int, sums_cached: bool) -> int:
    """Scalar ops to turn sum a'b' into an estimate of sum ab:
    2MN (s_a s_b D) + (MN + MZ) + (MN + NZ) + 2MN (Z m_a m_b) + 3MN (adds)
    = 9MN + MZ + NZ; with cached column sums the NZ term vanishes."""
    return 9 * M * N + M * Z + (0 if sums_cached else N * Z)


def quantized_mac_cost(M: int, N: int, Z: int) -> int:
    """Integer matmul cost 2MZN."""
    return 2 * M * Z * N


def decode_approximation_cost(d: int, L: int, sums_cached: bool = True) -> int:
    """Per decode iteration: QK^T (M=1, Z=d, N=L) + PV (M=1, Z=L, N=d)."""
    return approximation_cost(1, L, d, sums_cached) + approximation_cost(1, d, L, sums_cached)


def dequantization_cost(d: int, L: int) -> int:
    """Dequantize-first baseline: 2dL for K + 2dL for V = 4dL."""
    return 4 * d * L
