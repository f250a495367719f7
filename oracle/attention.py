"""HACK attention on quantized KV: prefill, decode (SE + RQE), exact attention.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows the paper's flow step by step (fig:overview; §5.3):
  (2) quantize Q (8-bit), K and V (b-bit) -- partition axes per
      fig:hoq_self_attn: Q and K along d_h; V along the sequence.
  (3) S = Q'K'^T by Eq. 4 per d_h-block, times 1/sqrt(d)
      (Eq. 2; reading R9: scale after Eq. 4).
  (4) P = softmax(S) row-wise (Eq. 3), causal in prefill (R8).
  (2) quantize P to 8 bits per (row, Pi-key block) aligned with V blocks
      (R6: round-to-nearest-even by default, R7).
  (3) O = P'V' by Eq. 4 per sequence block, plus the FP last block of V in full
      precision (RQE), no renormalisation (R14).
Decode: quantize k_new into its own partitions (R11),
append v_new to the FP16 tail, flush the tail when it reaches Pi (R12),
then attend with L_Q = 1.  Code sums are cached at quantization time (SE,
P:687) -- numerically identical to recomputing them.

Everything after code production is fp64; integer dot products are exact (an
fp64 GEMM over integers with |D| <= Pi*255*15 < 2^53 is exact).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import philox, quant
from .philox import TAG_K, TAG_Q


@dataclass
class Config:
    Hq: int
    Hkv: int
    d: int = 128
    Pi: int = 64
    bits: int = 2               # K/V code width b (Q and P are 8-bit)
    seed: int = 0x48414B
    layer: int = 0
    kv_round: str = "sr"
    q_round: str = "sr"
    p_round: str = "rn"         # reading R6 ("sr": the paper's stochastic rounding, selectable)
    head_base: int = 0          # global index of local KV head 0 (sharding)

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv

    @property
    def nbeta(self) -> int:
        return self.d // self.Pi

    def validate(self):
        if self.Hq % self.Hkv or self.d % self.Pi or self.bits not in (2, 4, 8):
            raise ValueError("bad config")


# ---------------------------------------------------------------- quantizers

def quantize_q(cfg: Config, q: np.ndarray, positions, rng_id: int):
    """Q [n, Hq, d] fp16 -> 8-bit codes [n,Hq,d], m/s fp32 [n,Hq,nb], sums [n,Hq,nb].
    Partitions along d_h, fp32 meta (transient, R4), SR by default (R6)."""
    n = q.shape[0]
    x = q.astype(np.float32).reshape(n, cfg.Hq, cfg.nbeta, cfg.Pi)
    u = None
    if cfg.q_round == "sr":
        u = np.empty((n, cfg.Hq, cfg.d), np.float32)
        for h in range(cfg.Hq):
            u[:, h] = philox.uniforms_rowwise(cfg.seed, rng_id, cfg.layer, TAG_Q,
                                              cfg.head_base * cfg.G + h, positions, cfg.d)
        u = u.reshape(x.shape)
    c, m, s, sm = quant.quantize(x, 8, "fp32", cfg.q_round, u)
    return c.reshape(n, cfg.Hq, cfg.d), m, s, sm


def quantize_k(cfg: Config, k: np.ndarray, positions, rng_id: int):
    """K [n, Hkv, d] fp16 -> b-bit codes, fp16 (m, s) [n,Hkv,nb], sums.  Each
    token forms its own partitions along d_h."""
    n = k.shape[0]
    x = k.astype(np.float32).reshape(n, cfg.Hkv, cfg.nbeta, cfg.Pi)
    u = None
    if cfg.kv_round == "sr":
        u = np.empty((n, cfg.Hkv, cfg.d), np.float32)
        for h in range(cfg.Hkv):
            u[:, h] = philox.uniforms_rowwise(cfg.seed, rng_id, cfg.layer, TAG_K,
                                              cfg.head_base + h, positions, cfg.d)
        u = u.reshape(x.shape)
    c, m, s, sm = quant.quantize(x, cfg.bits, "fp16", cfg.kv_round, u)
    return c.reshape(n, cfg.Hkv, cfg.d), m, s, sm


def quantize_v_block(cfg: Config, v_blk: np.ndarray, start: int, rng_id: int):
    """One full block of Pi tokens, V [Pi, Hkv, d] fp16 -> per (head, channel)
    partitions along the sequence: codes [Hkv, d, Pi], m/s/sums [Hkv, d]."""
    Pi = cfg.Pi
    assert v_blk.shape[0] == Pi
    x = np.transpose(v_blk.astype(np.float32), (1, 2, 0))          # [Hkv, d, Pi]
    u = None
    if cfg.kv_round == "sr":
        pos = np.arange(start, start + Pi)
        u = np.empty_like(x)
        for h in range(cfg.Hkv):
            u[h] = philox.uniforms_colwise(cfg.seed, rng_id, cfg.layer,
                                           cfg.head_base + h, pos, cfg.d).T
    return quant.quantize(x, cfg.bits, "fp16", cfg.kv_round, u)


def quantize_p(p_blk: np.ndarray, rnd: str = "rn", u: np.ndarray | None = None):
    """P partition = one row's Pi keys of one V block, 8-bit,
    transient fp64 meta.  Masked entries are exact zeros inside the partition
    (R8).  rnd: 'rn' round-to-nearest-even (the default reading R6) or 'sr' the
    paper's stochastic rounding (R1: floor(y) + [u < frac(y)]) with
    uniforms u of p_blk's shape.  Returns codes, m, s, sums, y (pre-rounding value,
    for the near-tie parity protocol)."""
    p = np.asarray(p_blk, np.float64)
    lo = p.min(-1)
    hi = p.max(-1)
    s = (hi - lo) / 255.0
    with np.errstate(divide="ignore", invalid="ignore"):
        y = (p - lo[..., None]) / s[..., None]
    y = np.where((s == 0)[..., None], 0.0, y)
    if rnd == "rn":
        c = np.rint(y)
    elif rnd == "sr":
        if u is None or np.shape(u) != p.shape:
            raise ValueError("stochastic rounding of P needs u with the partition's shape")
        fl = np.floor(y)
        c = fl + (np.asarray(u, np.float64) < (y - fl))
    else:
        raise ValueError(rnd)
    c = np.clip(c, 0, 255).astype(np.uint8)
    return c, lo, s, c.astype(np.int64).sum(-1), y


# ---------------------------------------------------------------- KV state

@dataclass
class KVState:
    """One request's quantized KV for one layer: K codes per token (partitions
    along d_h), committed V blocks (partitions along the sequence), FP16 tail
    (RQE), cached code sums (SE)."""
    cfg: Config
    rng_id: int = 0
    kc: list = field(default_factory=list)      # per token: codes [Hkv, d]
    km: list = field(default_factory=list)      # per token: m [Hkv, nb] (fp16 values)
    ks: list = field(default_factory=list)
    ksum: list = field(default_factory=list)
    vc: list = field(default_factory=list)      # per block: codes [Hkv, d, Pi]
    vm: list = field(default_factory=list)      # per block: m [Hkv, d]
    vs: list = field(default_factory=list)
    vsum: list = field(default_factory=list)
    tail: list = field(default_factory=list)    # fp16 rows [Hkv, d], < Pi of them

    @property
    def length(self) -> int:
        return len(self.kc)

    @property
    def nblocks(self) -> int:
        return len(self.vc)

    def append_k(self, k_rows: np.ndarray):
        pos = np.arange(self.length, self.length + k_rows.shape[0])
        c, m, s, sm = quantize_k(self.cfg, k_rows, pos, self.rng_id)
        for i in range(k_rows.shape[0]):
            self.kc.append(c[i]); self.km.append(m[i]); self.ks.append(s[i]); self.ksum.append(sm[i])

    def append_v(self, v_row: np.ndarray):
        """Append one token's V to the FP16 tail; flush exactly when it reaches
        Pi tokens.  Committed blocks are never touched again (RQE)."""
        self.tail.append(np.asarray(v_row, np.float16))
        if len(self.tail) == self.cfg.Pi:
            start = self.nblocks * self.cfg.Pi
            c, m, s, sm = quantize_v_block(self.cfg, np.stack(self.tail), start, self.rng_id)
            self.vc.append(c); self.vm.append(m); self.vs.append(s); self.vsum.append(sm)
            self.tail = []

    def arrays(self):
        """Stacked views: K codes [L,Hkv,d], km/ks/ksum [L,Hkv,nb]; V codes
        [nb,Hkv,d,Pi], vm/vs/vsum [nb,Hkv,d]; tail [T,Hkv,d] fp16."""
        cfg = self.cfg
        st = lambda a, shp, dt: np.stack(a) if a else np.zeros((0,) + shp, dt)
        return dict(
            kc=st(self.kc, (cfg.Hkv, cfg.d), np.uint8),
            km=st(self.km, (cfg.Hkv, cfg.nbeta), np.float32),
            ks=st(self.ks, (cfg.Hkv, cfg.nbeta), np.float32),
            ksum=st(self.ksum, (cfg.Hkv, cfg.nbeta), np.int64),
            vc=st(self.vc, (cfg.Hkv, cfg.d, cfg.Pi), np.uint8),
            vm=st(self.vm, (cfg.Hkv, cfg.d), np.float32),
            vs=st(self.vs, (cfg.Hkv, cfg.d), np.float32),
            vsum=st(self.vsum, (cfg.Hkv, cfg.d), np.int64),
            tail=st(self.tail, (cfg.Hkv, cfg.d), np.float16),
        )


def ingest_prompt(cfg: Config, k: np.ndarray, v: np.ndarray, rng_id: int = 0) -> KVState:
    """Quantize a prompt's K/V: every token's K, every full Pi-token V
    block; the ragged V remainder stays FP16 (reading R10)."""
    cfg.validate()
    st = KVState(cfg, rng_id)
    st.append_k(k)
    for t in range(v.shape[0]):
        st.append_v(v[t])
    return st


# ---------------------------------------------------------------- attention core

def _attend(cfg: Config, st: dict, qc, qm, qs, qsum, pos, hq, pcodes_override=None, rng_id: int = 0):
    """Rows of one query head hq against the state's keys 0..L-1, each row i
    seeing keys t <= pos[i].  Returns O [n, d] fp64 and diagnostics."""
    d, Pi, nb = cfg.d, cfg.Pi, cfg.nbeta
    hk = hq // cfg.G
    L = st["kc"].shape[0]
    n = qc.shape[0]
    kc = st["kc"][:, hk, :].astype(np.float64)                 # [L, d]
    # (3) Eq. 4 per d_h block, then 1/sqrt(d) (R9)
    S = np.zeros((n, L), np.float64)
    for beta in range(nb):
        sl = slice(beta * Pi, (beta + 1) * Pi)
        D = np.rint(qc[:, sl].astype(np.float64) @ kc[:, sl].T)  # exact integers
        sa = qs[:, beta].astype(np.float64)[:, None]
        ma = qm[:, beta].astype(np.float64)[:, None]
        SA = qsum[:, beta].astype(np.float64)[:, None]
        sb = st["ks"][:, hk, beta].astype(np.float64)[None, :]
        mb = st["km"][:, hk, beta].astype(np.float64)[None, :]
        SB = st["ksum"][:, hk, beta].astype(np.float64)[None, :]
        S += sa * sb * D + mb * sa * SA + ma * sb * SB + Pi * ma * mb
    S /= np.sqrt(d)
    # (4) causal softmax (Eq. 3, R8)
    visible = np.arange(L)[None, :] <= np.asarray(pos)[:, None]
    S = np.where(visible, S, -np.inf)
    S = S - S.max(axis=1, keepdims=True)
    E = np.where(visible, np.exp(S), 0.0)
    P = E / E.sum(axis=1, keepdims=True)
    # (2)+(3) P quantization per committed V block, Eq. 4 for P V
    O = np.zeros((n, d), np.float64)
    nfull = st["vc"].shape[0]
    py = np.zeros((n, nfull * Pi))
    pcodes = np.zeros((n, nfull * Pi), np.uint8)
    pu = None
    if cfg.p_round == "sr" and nfull:   # position-keyed P stream of this query head (R3)
        pu = philox.uniforms_p(cfg.seed, rng_id, cfg.layer, cfg.head_base * cfg.G + hq, pos, np.arange(nfull * Pi))
    for j in range(nfull):
        sl = slice(j * Pi, (j + 1) * Pi)
        c, m_p, s_p, SP, y = quantize_p(P[:, sl], cfg.p_round, None if pu is None else pu[:, sl])
        if pcodes_override is not None:
            c = np.asarray(pcodes_override[:, sl], np.uint8)
            SP = c.astype(np.int64).sum(-1)
        py[:, sl] = y
        pcodes[:, sl] = c
        vc = st["vc"][j, hk].astype(np.float64)                # [d, Pi]
        Dp = np.rint(c.astype(np.float64) @ vc.T)              # [n, d] exact
        sv = st["vs"][j, hk].astype(np.float64)[None, :]
        mv = st["vm"][j, hk].astype(np.float64)[None, :]
        SV = st["vsum"][j, hk].astype(np.float64)[None, :]
        sp, mp, SPc = s_p[:, None], m_p[:, None], SP.astype(np.float64)[:, None]
        O += sp * sv * Dp + mv * sp * SPc + mp * sv * SV + Pi * mp * mv
    # FP16 last block of V in full precision (RQE)
    T = L - nfull * Pi
    if T:
        O += P[:, nfull * Pi:] @ st["tail"][:T, hk, :].astype(np.float64)
    return O, dict(P=P, pcodes=pcodes, py=py, pu=pu)


def prefill(cfg: Config, q: np.ndarray, k: np.ndarray, v: np.ndarray, rng_id: int = 0,
            rows=None, heads=None, pcodes_override=None, keep_diag=False):
    """HACK prefill for one request: returns (O [L,Hq,d] fp64,
    KVState, diagnostics).  `rows` / `heads` restrict which outputs are
    computed (sampled parity at full size); other rows are NaN."""
    cfg.validate()
    L = q.shape[0]
    state = ingest_prompt(cfg, k, v, rng_id)
    st = state.arrays()
    rows = np.arange(L) if rows is None else np.asarray(rows)
    heads = range(cfg.Hq) if heads is None else heads
    qc, qm, qs, qsum = quantize_q(cfg, q[rows], rows, rng_id)
    O = np.full((L, cfg.Hq, cfg.d), np.nan)
    diag = {}
    for hq in heads:
        ov = None if pcodes_override is None else pcodes_override[hq]
        o, dg = _attend(cfg, st, qc[:, hq], qm[:, hq], qs[:, hq], qsum[:, hq], rows, hq, ov, rng_id)
        O[rows, hq] = o
        if keep_diag:
            diag[hq] = dg
    return O, state, diag


def decode_step(state: KVState, q_new: np.ndarray, k_new: np.ndarray, v_new: np.ndarray,
                keep_diag=False):
    """One decode iteration for one request: quantize and append
    k_new (own partitions), append v_new to the FP16 tail and flush at
    Pi, then attend with L_Q = 1 over every cached token.
    q_new [Hq, d], k_new/v_new [Hkv, d] fp16.  Returns O [Hq, d] fp64."""
    state.append_k(k_new[None])
    state.append_v(v_new)
    return decode_attend(state, q_new, keep_diag=keep_diag)


def decode_attend(state: KVState, q_new: np.ndarray, pcodes_override=None, keep_diag=False):
    """The attention half of decode_step: q_new (position length-1) over every cached
    token of the state as it stands.  `pcodes_override` {hq: [1, committed]} replaces
    the P codes (near-tie protocol)."""
    cfg = state.cfg
    pos = state.length - 1
    st = state.arrays()
    qc, qm, qs, qsum = quantize_q(cfg, q_new[None], np.array([pos]), state.rng_id)
    O = np.zeros((cfg.Hq, cfg.d))
    diag = {}
    for hq in range(cfg.Hq):
        ov = None if pcodes_override is None else pcodes_override.get(hq)
        o, dg = _attend(cfg, st, qc[:, hq], qm[:, hq], qs[:, hq], qsum[:, hq], [pos], hq, ov, state.rng_id)
        O[hq] = o[0]
        if keep_diag:
            diag[hq] = dg
    return O, diag


# ---------------------------------------------------------------- exact reference

def exact_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, causal: bool = True,
                    q_positions=None) -> np.ndarray:
    """Eq. 2-3 in fp64 with no quantization (O9), GQA by head
    grouping (R15).  q [n,Hq,d], k/v [L,Hkv,d] -> O [n,Hq,d]."""
    n, Hq, d = q.shape
    L, Hkv, _ = k.shape
    G = Hq // Hkv
    pos = np.arange(L - n, L) if q_positions is None else np.asarray(q_positions)
    O = np.zeros((n, Hq, d))
    for hq in range(Hq):
        hk = hq // G
        S = q[:, hq].astype(np.float64) @ k[:, hk].astype(np.float64).T / np.sqrt(d)
        if causal:
            S = np.where(np.arange(L)[None, :] <= pos[:, None], S, -np.inf)
        S = S - S.max(axis=1, keepdims=True)
        E = np.exp(S)
        O[:, hq] = (E / E.sum(axis=1, keepdims=True)) @ v[:, hk].astype(np.float64)
    return O
