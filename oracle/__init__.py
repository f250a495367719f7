"""CPU oracle for HACK (arXiv 2502.03589) -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference the CUDA path is
checked against.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product package
(`paper_2502_03589_b200`) never imports it and has no CPU fallback.

It shares no code with the CUDA path: its own Philox4x32-10, its own
quantizer, its own page packer, fp64 Eq. 4 / softmax / outputs.  Citations are
`P:<line>` = /root/reference/PAPER.md line, `S:<line>` = SPEC.md line.

Modules
  philox    Philox4x32-10 counter-based RNG and the position-keyed counter map.
  quant     per-partition asymmetric b-bit quantizer, pack/unpack.
  homomm    Eq. 4 homomorphic matmul + dequantize-then-multiply twin + cost model.
  attention HACK prefill / decode (SE, RQE), exact attention (Eq. 2-3).
  pages     the paged packed-KV layout of DESIGN.md "HBM layout" (bytes).

Parity pins: every function is pinned by tests/test_oracle_*.py against values
the paper/SPEC fix (worked examples in tests/golden), closed forms, invariants,
brute force.  No function here is "parity unpinned".
"""
from . import philox, quant, homomm, attention, pages  # noqa: F401
