"""Property-based checks (hypothesis) of the host-side logic against the oracle: the
C-ABI chunk partition and byte accounting, the rate schedule, the ring plan, config
resolution and RunTrace invariants.  CPU only (the library's host functions load
without a GPU)."""

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import lasgd_oracle as O
from paper_2203_13085_b200 import cli
from paper_2203_13085_b200 import problems as PR
from paper_2203_13085_b200.collective import bytes_per_node, ring_schedule
from paper_2203_13085_b200.params import partition_chunks
from paper_2203_13085_b200.trace import RoundRecord, RunTrace

SETTINGS = settings(max_examples=200, deadline=None)


@SETTINGS
@given(st.integers(1, 10**7), st.integers(1, 8))
def test_partition_matches_oracle_and_is_balanced(d, P):
    got = [tuple(b) for b in partition_chunks(d, P).bounds]
    assert got == O.partition_chunks(d, P)
    sizes = [e - s for s, e in got]
    assert sum(sizes) == d and max(sizes) - min(sizes) <= 1 and got[0][0] == 0 and got[-1][1] == d
    assert all(got[i][1] == got[i + 1][0] for i in range(P - 1))


@SETTINGS
@given(st.integers(1, 10**7), st.integers(1, 8), st.sampled_from([2, 4, 8]),
       st.one_of(st.none(), st.integers(0, 7)))
def test_bytes_per_node_matches_oracle(d, P, bpe, rank):
    if rank is not None and rank >= P:
        rank = P - 1
    assert bytes_per_node(d, P, bpe, rank) == O.bytes_per_node(d, P, bpe, rank)


@SETTINGS
@given(st.integers(1, 8))
def test_ring_schedule_shape(P):
    sched = ring_schedule(P)
    assert sched.num_steps == 2 * (P - 1)
    for step in sched.steps:
        assert sorted(s.send_chunk for s in step) == list(range(P))  # every chunk moves once per step
        assert all(s.send_to == (r + 1) % P and s.recv_from == (r - 1) % P for r, s in enumerate(step))


@SETTINGS
@given(st.floats(1e-4, 1.0), st.integers(1, 64), st.floats(0, 10), st.lists(st.floats(0, 100), max_size=3),
       st.floats(1.5, 20), st.integers(1, 500), st.integers(0, 100_000))
def test_lr_schedule_matches_oracle(base, scale, warm, decays, factor, spe, step):
    a = PR.lr_at(PR.LrSchedule(base, scale, warm, tuple(decays), factor, spe), step)
    b = O.lr_at(O.LrSchedule(base, scale, warm, tuple(decays), factor, spe), step)
    assert a == b


@SETTINGS
@given(st.integers(1, 8), st.floats(0.01, 1.0), st.sampled_from(["pull", "delta"]), st.booleans(),
       st.integers(1, 1000), st.integers(1, 512))
def test_config_resolution_is_idempotent(tau, alpha, mode, adaptive, steps, batch):
    raw = {"lasgd": {"tau_max": tau, "alpha": 1.0 if mode == "delta" else alpha, "mode": mode,
                     "adaptive": adaptive}, "steps": steps, "problem": {"batch": batch}}
    cfg = cli.resolve(raw)
    assert cli.resolve(cfg) == cfg
    assert cli.config_hash(cli.resolve(cfg)) == cli.config_hash(cfg)


@SETTINGS
@given(st.integers(1, 6), st.integers(1, 40), st.data())
def test_runtrace_invariants_hold_for_any_round_pattern(P, rounds, data):
    per_rank = []
    for _ in range(P):
        k = data.draw(st.integers(0, rounds))
        clock, t, recs = 0, 0.0, []
        for i in range(k):
            tau = data.draw(st.integers(1, 5))
            clock += tau
            t += data.draw(st.floats(1e-6, 1.0))
            recs.append(RoundRecord(i + 1, clock, tau, 0.1, t, None))
        per_rank.append(recs)
    tr = RunTrace(per_rank, 1000)
    tr.validate()
    rows = tr.rows()
    assert len(rows) == max(len(r) for r in per_rank)
    if rows:
        assert rows[-1]["bytes_sent"] == tr.rounds * (bytes_per_node(1000, P, 4) if P > 1 else 0)
        assert rows[-1]["grad_evals"] == sum(r[-1].local_clock for r in per_rank if r)


def test_ring_mean_order_property():
    """The ring order is a rotation per chunk: chunk c starts at rank c (collective.py:183-200)."""
    rng = np.random.default_rng(0)
    P, n = 5, 23
    vecs = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    got = O.ring_mean(vecs)
    for c, (s, e) in enumerate(O.partition_chunks(n, P)):
        acc = vecs[c][s:e].copy()
        for k in range(1, P):
            acc = acc + vecs[(c + k) % P][s:e]
        assert np.array_equal(got[s:e], acc / np.float32(P))


def test_degenerate_inputs_raise_like_the_reference():
    """params.py:39,55,136-139: zero-dimension vectors and zero chunk counts are
    ValueErrors; d < num_chunks gives trailing empty ranges at offset d."""
    import pytest
    import torch

    from paper_2203_13085_b200.params import as_device_vector

    with pytest.raises(ValueError, match="positive dimension"):
        as_device_vector(np.zeros(0), device=torch.device("cpu"))
    with pytest.raises(ValueError, match="1-D"):
        as_device_vector(np.float64(1.0), device=torch.device("cpu"))
    with pytest.raises(ValueError, match="d must be positive"):
        partition_chunks(0, 3)
    with pytest.raises(ValueError, match="num_chunks must be positive"):
        partition_chunks(5, 0)
    assert [tuple(b) for b in partition_chunks(2, 5).bounds] == [(0, 1), (1, 2), (2, 2), (2, 2), (2, 2)]


def test_sgd_ar_bucket_plan_covers_the_vector_in_reverse():
    """BucketedSGDARWorker's buckets: contiguous, disjoint, cover [0, n) from the end,
    16-byte aligned boundaries, at most bucket_bytes each; every tensor is counted in
    every bucket it overlaps (CPU, no device)."""
    import random

    from paper_2203_13085_b200.engine import plan_buckets

    rng = random.Random(3)
    for _ in range(200):
        sizes = [rng.randint(1, 5000) for _ in range(rng.randint(1, 30))]
        align = rng.choice([1, 64])
        offs, off = [], 0
        for c in sizes:
            off = (off + align - 1) // align * align
            offs.append(off)
            off += c
        n = off
        bb = rng.choice([16, 100, 4096, 40_000, 1 << 30])
        buckets, member, need = plan_buckets(n, list(zip(offs, sizes)), bb, 4)
        assert buckets[0][1] == n and buckets[-1][0] == 0
        for (lo, hi), (lo2, hi2) in zip(buckets, buckets[1:]):
            assert hi2 == lo and lo2 < hi2
        for lo, hi in buckets:
            assert lo % 4 == 0 and 0 < hi - lo <= max(4, bb // 4 // 4 * 4) + 3
        for b in range(len(buckets)):
            lo, hi = buckets[b]
            assert need[b] == sum(1 for o, c in zip(offs, sizes) if o < hi and lo < o + c)
        for (o, c), bs in zip(zip(offs, sizes), member):
            assert bs and all(buckets[b][0] < o + c and o < buckets[b][1] for b in bs)
