"""Host logic of the C5 disaggregated-trace driver (bench_c5.py), no GPU: the synthetic trace
follows tab:dataset and Poisson arrivals; the schedule assigns by shortest
queue."""
import numpy as np

import bench_c5


def test_length_mixture_matches_the_dataset_table():
    rng = np.random.default_rng(1)
    for name, ((pm, plo, phi), (om, olo, ohi)) in bench_c5.DATASETS.items():
        p = bench_c5.lognormal_clipped(rng, pm, plo, phi, 40000)
        o = bench_c5.lognormal_clipped(rng, om, olo, ohi, 40000)
        assert p.min() >= plo and p.max() <= phi and o.min() >= olo and o.max() <= ohi
        assert abs(p.mean() / pm - 1) < 0.03, name          # clipping at ~1/99 pct barely moves the mean
        assert abs(o.mean() / om - 1) < 0.08, name


def test_poisson_arrivals_and_caps():
    tr = bench_c5.make_trace(4000, 50.0, 7, max_prompt=8192, max_output=100)
    gaps = np.diff([r["arrival"] for r in tr])
    assert abs(gaps.mean() * 50.0 - 1) < 0.05                # exponential gaps at rate 50
    assert abs(np.std(gaps) / np.mean(gaps) - 1) < 0.08      # CV of an exponential = 1
    assert max(r["prompt"] for r in tr) <= 8192 and max(r["output"] for r in tr) <= 100
    assert {r["dataset"] for r in tr} == set(bench_c5.DATASETS)
    assert bench_c5.make_trace(50, 1.0, 7, 8192, 100) == bench_c5.make_trace(50, 1.0, 7, 8192, 100)  # seeded


def test_shortest_queue_schedule():
    tr = bench_c5.make_trace(400, 1.0, 3, 16384, 256)
    for r in tr:
        r["arrival"] *= 1e-4          # a burst: queues build up
    bench_c5.schedule(tr, 4, 4, pre_tok_s=1e6)
    # prefill: every request went to a rank whose modelled queue was shortest at its arrival
    free = [0.0] * 4
    for r in tr:
        start = [max(f, r["arrival"]) for f in free]
        assert start[r["pre"]] == min(start)
        free[r["pre"]] = start[r["pre"]] + r["prompt"] / 1e6
    # decode: assigned tokens balanced to within one request's tokens
    load = np.zeros(4)
    for r in tr:
        load[r["dec"]] += r["prompt"] + r["output"]
    assert load.max() - load.min() <= max(r["prompt"] + r["output"] for r in tr)
