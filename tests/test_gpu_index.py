"""GPU parity of the device n-gram index (store.cuh): the indexed lookup == the scanning lookup == the
oracle (a restatement of datastore.cpp:49-132, itself pinned to the reference's golden vectors), on
the reference-generated lookup cases and on a paper-scale prior (~9.5 MB of tokens)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1, "no sm_100 device / library failed to load"
    return dbl


def _store(dbl, max_order, rej, inserts, index_after=None):
    st = dbl.HierarchicalDatastore(max_order, 10)
    st.rejected_enabled = rej
    layers = (st.prior, st.dynamic, st.rejected)
    for i, (layer, toks, step) in enumerate(inserts):
        if index_after is not None and i == index_after:
            for ly in layers:
                ly.build_index()
        layers[layer].insert(toks, step)
    if index_after is None:
        for ly in layers:
            ly.build_index()
    return st


def test_index_golden_vectors(dbl):
    """Every reference-generated lookup case, with every layer indexed, and with an index over the first
    half of the inserts plus a scanned tail."""
    cases = json.load(open(os.path.join(GOLDEN, "lookups.json")))
    for case in cases:
        for split in (None, len(case["inserts"]) // 2):
            st = _store(dbl, case["max_order"], case["rejected_enabled"], case["inserts"], split)
            got = [[r.candidates, r.source, r.matched_order] for r in (st.lookup(c, d) for c, d in case["queries"])]
            assert got == case["results"], (case, split)
            s = st.stats
            assert [s.lookups, s.prior_hits, s.dynamic_hits, s.rejected_hits, s.fallback_hits, s.misses] == case["stats"]


def test_index_known_answers(dbl):
    # test_datastore.cpp:62-136 through an indexed prior
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, [[1, 2, 3, 4, 5, 6]], 1)  # small priors are scanned (index past 4,096 tokens)
    assert st.prior.index_entries == 0
    st.prior.build_index()
    assert st.prior.index_entries > 0
    r = st.lookup([9, 2, 3], 10)
    assert (r.candidates, r.source, r.matched_order) == ([4, 5, 6], "prior", 2)
    st = dbl.HierarchicalDatastore(3, 3)
    dbl.build_prior(st, [[1, 2, 3, 4, 5, 6, 7, 8]], 1)
    st.prior.build_index()
    assert st.lookup([1, 2], 3).candidates == [3, 4, 5]
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, [[5, 6, 7, 1], [7, 2, 3]], 2)  # higher order beats layer / recency
    st.prior.build_index()
    st.dynamic.insert([1, 2, 3, 9], 5)
    r = st.lookup([7, 2, 3], 10)  # (7,2,3) and the prior's (2,3) end their sequence: avail 0, skipped
    assert (r.candidates, r.source, r.matched_order) == ([9], "dynamic", 2)


def _stream(vocab, n, seed, rho=0.9):
    rng = np.random.default_rng(seed)
    s = list(rng.integers(1, vocab - 1, 8))
    while len(s) < n:
        if rng.random() < rho:
            span = int(rng.integers(4, 17))
            st = int(rng.integers(0, len(s)))
            s.extend(s[st:st + span])
        else:
            s.extend(int(x) for x in rng.integers(1, vocab - 1, int(rng.integers(1, 5))))
    return s[:n]


def test_paper_scale_prior(dbl):
    """~2.4 M tokens (9.6 MB int32: the paper's K = 10 prior is ~9.5 MB) built with build_prior (device
    index), a dynamic and a rejected layer on top; 120 lookups == the oracle's scan; the indexed lookup
    is timed against a full scan of the same store."""
    from oracle.pyoracle import Oracle
    V, seq_len, n_seq = 151936, 64, 37500
    flat = _stream(V, seq_len * n_seq, 7)
    seqs = [flat[i * seq_len:(i + 1) * seq_len] for i in range(n_seq)]
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, seqs, n_seq)
    assert st.prior.index_entries > 2 * len(flat)
    orc = Oracle().store(3, 10)
    for i, q in enumerate(seqs):
        orc.insert(0, q, i)
    rng = np.random.default_rng(3)
    extra = [(1, _stream(V, 70, 11), 40000), (2, _stream(V, 50, 12), 40001), (1, flat[5000:5060], 40002)]
    for layer, toks, step in extra:
        (st.prior, st.dynamic, st.rejected)[layer].insert(toks, step)
        orc.insert(layer, toks, step)
    queries = []
    for k in range(120):
        if k % 6 == 5:  # random context: mostly misses / fallback
            ctx = [int(x) for x in rng.integers(1, V - 1, int(rng.integers(1, 12)))]
        else:
            a = int(rng.integers(0, len(flat) - 40))
            ctx = flat[a:a + int(rng.integers(1, 40))]
            if k % 4 == 3:
                ctx = ctx + [int(rng.integers(1, V - 1))]  # order 1/2 only
        queries.append((ctx, int(rng.integers(1, 12))))
    for ctx, d in queries:
        got = st.lookup(ctx, d)
        want = orc.lookup(ctx, d)
        assert (got.candidates, got.source, got.matched_order) == want, (ctx, d)
    # timing: the index vs a scan of the same content (an unindexed copy of the prior)
    ctx = flat[123456:123476]
    us_idx = st.profile_lookup(ctx, 10, 200)
    scan = dbl.HierarchicalDatastore(3, 10)
    for i in range(0, n_seq, 500):  # appended, not bulk-loaded: no index
        for j, q in enumerate(seqs[i:i + 500]):
            scan.prior.insert(q, i + j)
    assert scan.prior.index_entries == 0
    assert scan.lookup(ctx, 10).candidates == st.lookup(ctx, 10).candidates
    us_scan = scan.profile_lookup(ctx, 10, 20)
    print(f"paper-scale prior ({len(flat)} tokens): indexed lookup {us_idx:.1f} us, full scan {us_scan:.1f} us")
    assert us_idx < us_scan
