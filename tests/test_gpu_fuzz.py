"""GPU parity over seeded random configurations (prefill + decode) vs the oracle.

Each case draws (Pi, b, G, H_kv, prompt lengths, decode steps, rounding) from a fixed
seed, so the set is reproducible.  The draws cover the shapes the hand-picked tests miss,
e.g. Pi = 32 with G = 3 or Pi = 128 with ragged multi-request batches.  The bar is the
parity protocol used everywhere else: pages bit-exact; outputs <= 1e-3 row-relative;
P-code mismatches only at near-ties."""
import numpy as np
import pytest

from oracle import attention as att

from .test_gpu_decode import run_decode
from .test_gpu_prefill import check_request, run_prefill

pytestmark = pytest.mark.gpu


def draw(case):
    rng = np.random.default_rng(31337 + case)
    Pi = int(rng.choice([32, 64, 128]))
    bits = int(rng.choice([2, 4]))
    G = int(rng.choice([1, 2, 3, 4, 6, 8]))
    Hkv = int(rng.choice([1, 2]))
    n = int(rng.integers(1, 4))
    prompts = [int(x) for x in rng.integers(1, 3 * Pi + 7, n)]
    steps = int(rng.integers(2, Pi + 3))
    kv_round = "rn" if case % 5 == 4 else "sr"
    return att.Config(Hq=G * Hkv, Hkv=Hkv, Pi=Pi, bits=bits, seed=int(rng.integers(1, 1 << 30)),
                      kv_round=kv_round, layer=int(rng.integers(0, 4))), prompts, steps


@pytest.mark.parametrize("case", range(24))
def test_random_prefill(case):
    ocfg, prompts, _ = draw(case)
    print(ocfg, prompts)
    res = run_prefill(ocfg, prompts, seed=100 + case)
    for i in range(len(prompts)):
        check_request(ocfg, i, *res)


@pytest.mark.parametrize("case", range(24))
def test_random_decode(case):
    ocfg, prompts, steps = draw(case)
    print(ocfg, prompts, steps)
    run_decode(ocfg, prompts, steps, seed=200 + case, check_every=max(1, steps // 4))
