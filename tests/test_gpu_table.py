"""GPU parity: retrieval kernel + the full device DOUBLE loop on table models (config 1 and the
reference's acceptance set) against golden vectors produced by the unmodified reference.
Bit-exact: outputs, traces_to_jsonl text (sha256), metrics, lookup results and stats."""
import hashlib
import json
import os
import random

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CFG1 = json.load(open(os.path.join(GOLDEN, "config1.json")))


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1, "no sm_100 device / library failed to load"
    return dbl


def _store(dbl, max_order, rej, inserts):
    st = dbl.HierarchicalDatastore(max_order, 10)
    st.rejected_enabled = rej
    for layer, toks, step in inserts:
        (st.prior, st.dynamic, st.rejected)[layer].insert(toks, step)
    return st


def test_lookup_golden_vectors_single_and_batch(dbl):
    cases = json.load(open(os.path.join(GOLDEN, "lookups.json")))
    for case in cases:
        st = _store(dbl, case["max_order"], case["rejected_enabled"], case["inserts"])
        got = [[r.candidates, r.source, r.matched_order]
               for r in (st.lookup(c, d) for c, d in case["queries"])]
        assert got == case["results"]
        s = st.stats
        assert [s.lookups, s.prior_hits, s.dynamic_hits, s.rejected_hits, s.fallback_hits,
                s.misses] == case["stats"]
        st2 = _store(dbl, case["max_order"], case["rejected_enabled"], case["inserts"])
        got2 = st2.lookup_batch([c for c, _ in case["queries"]], [d for _, d in case["queries"]])
        assert [[r.candidates, r.source, r.matched_order] for r in got2] == case["results"]


def test_lookup_known_answers(dbl):
    # test_datastore.cpp:62-172 restated against the device store
    st = dbl.HierarchicalDatastore(3, 10)
    st.prior.insert([1, 2, 3, 4, 5, 6], 0)
    r = st.lookup([9, 2, 3], 10)
    assert (r.candidates, r.source, r.matched_order) == ([4, 5, 6], "prior", 2)
    st = dbl.HierarchicalDatastore(3, 10)
    st.prior.insert([1, 2, 3, 4, 5, 6, 7, 8], 0)
    assert st.lookup([1, 2], 3).candidates == [3, 4, 5]
    assert st.lookup([1, 2], 100).candidates == [3, 4, 5, 6, 7, 8]
    st = dbl.HierarchicalDatastore(2, 10)
    st.dynamic.insert([1, 2, 5], 0)
    st.dynamic.insert([1, 2, 6], 3)
    st.dynamic.insert([1, 2, 4], 1)
    assert st.lookup([1, 2], 10).candidates == [6]
    st = dbl.HierarchicalDatastore(3, 10)
    r = st.lookup([1, 2, 9, 1, 2, 8, 1, 2], 10)
    assert (r.candidates, r.source, r.matched_order) == ([8, 1, 2], "context", 2)
    r = st.lookup([5, 1, 2, 3, 7, 1, 2, 3], 2)
    assert (r.matched_order, r.candidates) == (3, [7, 1])
    assert st.lookup([1, 2, 3], 10).source == "miss"
    with pytest.raises(dbl.InvalidArgument):
        st.lookup([], 10)
    with pytest.raises(dbl.InvalidArgument):
        st.prior.insert([], 0)
    st = dbl.HierarchicalDatastore(2, 10)
    st.record_accepted([1, 2, 5])
    st.record_rejected([1, 2, 6])
    st.record_accepted([])
    assert st.lookup([1, 2], 10).source == "dynamic"
    st.flush_session()
    assert st.lookup([1, 2], 10).source == "miss"
    assert st.dynamic.sequences == [] and st.rejected.sequences == []
    assert st.step_counter == 2


def test_lookup_fuzz_vs_oracle_large_store(dbl, oracle):
    """Big layers (multi-thousand tokens) exercise the strided CTA scan and the reductions."""
    rng = random.Random(5)
    for trial in range(6):
        mo = rng.choice([2, 3, 4])
        V = rng.choice([4, 8, 50])
        ins = [(rng.choice([0, 1, 2]), [rng.randrange(V) for _ in range(rng.randint(1, 400))],
                rng.randint(0, 50)) for _ in range(40)]
        st = _store(dbl, mo, True, ins)
        o = oracle.store(mo, 10)
        for l, t, s in ins:
            o.insert(l, t, s)
        qs = [([rng.randrange(V) for _ in range(rng.randint(1, 60))], rng.choice([1, 5, 10, 64]))
              for _ in range(50)]
        got = st.lookup_batch([q for q, _ in qs], [d for _, d in qs])
        for (q, d), g in zip(qs, got):
            assert [g.candidates, g.source, g.matched_order] == list(o.lookup(q, d))
        assert len(st.prior.sequences) == sum(1 for l, _, _ in ins if l == 0)


def _config1_models(dbl):
    d = dbl.TableModel.from_model_v1(open(os.path.join(GOLDEN, "config1_draft.model-v1")).read())
    t = dbl.TableModel.from_model_v1(open(os.path.join(GOLDEN, "config1_target.model-v1")).read())
    return d, t


def _config1_store(dbl, rejected=True):
    from paper_2601_05524_b200.specpar import parse_dstore_v1
    mo, seqs = parse_dstore_v1(open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read())
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, seqs, len(seqs))
    st.rejected_enabled = rejected
    return st


@pytest.mark.parametrize("method", ["double", "psd", "target_retrieval", "draft_retrieval", "sd",
                                    "vanilla_ar"])
def test_config1_bit_exact(dbl, method):
    d, t = _config1_models(dbl)
    prompt = CFG1["prompt"]
    want = CFG1["methods"][method]
    opts = dbl.PipelineOptions(gamma=2, depth=10, t_target=1.0, t_draft=0.625)
    if method == "vanilla_ar":
        r = dbl.run_vanilla_ar(t, prompt, 256, t_target=1.0)
    elif method in ("sd", "draft_retrieval"):
        r = dbl.run_serial_sd(d, t, _config1_store(dbl), prompt, 256, opts,
                              use_retrieval=method == "draft_retrieval")
    else:
        opts.draft_retrieval = method == "double"
        opts.target_retrieval = method in ("double", "target_retrieval")
        r = dbl.run(d, t, _config1_store(dbl), prompt, 256, opts)
    assert r.output == want["output"]
    assert sha(r.jsonl) == want["jsonl_sha256"], (r.jsonl.splitlines()[:3], want.get("jsonl", "")[:400])
    m = want["metrics"]
    got = r.metrics
    assert [got["tokens"], got["rounds"], got["clock"], got["m"], got["amt"], got["speedup"],
            got["hit_rate"], got["lookups"]] == [m[k] for k in
                                                 ("tokens", "rounds", "clock", "m", "amt", "speedup",
                                                  "hit_rate", "lookups")]


def test_acceptance_set_on_device(dbl, oracle):
    """The reference's criterion-1 set (acceptance.cpp:62-125): device DOUBLE == golden reference
    traces, and == target-only greedy AR."""
    acc = json.load(open(os.path.join(GOLDEN, "acceptance100.json")))
    for case in acc[:40]:
        c = case["config"]
        corpus = oracle.gen_corpus(c["vocab"], c["rho"], c["corpus_len"], c["seed"])
        dm = dbl.TableModel.from_model_v1(oracle.table_build(corpus, c["draft_order"], 0.1, c["vocab"]).serialize())
        tm = dbl.TableModel.from_model_v1(oracle.table_build(corpus, c["target_order"], 0.1, c["vocab"]).serialize())
        st = dbl.HierarchicalDatastore(3, c["depth"])
        dbl.build_prior(st, corpus, 10)
        opts = dbl.PipelineOptions(gamma=c["gamma"], depth=c["depth"])
        r = dbl.run(dm, tm, st, corpus[0][:8], 256, opts)
        assert sha(" ".join(map(str, r.output))) == case["output_sha256"]
        assert sha(r.jsonl) == case["jsonl_sha256"]
        ar = dbl.run_vanilla_ar(tm, corpus[0][:8], 256)
        assert ar.output == r.output


def test_forward_batch_rows_match_oracle(dbl, oracle):
    d, t = _config1_models(dbl)
    ot = oracle.table_parse(open(os.path.join(GOLDEN, "config1_target.model-v1")).read())
    rng = random.Random(1)
    for _ in range(30):
        ctx = [rng.randrange(32) for _ in range(rng.randint(1, 20))]
        cands = [rng.randrange(32) for _ in range(rng.randint(0, 12))]
        assert dbl.forward_batch(t, ctx, cands) == ot.argmax_rows(ctx, cands)
    with pytest.raises(dbl.InvalidArgument):
        dbl.forward_batch(t, [], [1])


def test_pipeline_errors_map_to_reference_types(dbl):
    d, t = _config1_models(dbl)
    st = _config1_store(dbl)
    with pytest.raises(dbl.InvalidArgument):
        dbl.run(d, t, st, [], 10)
    with pytest.raises(dbl.InvalidArgument):
        dbl.run(d, t, st, [1, 2], 0)
    with pytest.raises(dbl.InvalidArgument):
        dbl.run(d, t, st, [1, 2], 10, dbl.PipelineOptions(gamma=0))
    with pytest.raises(dbl.InvalidArgument):
        dbl.run(d, t, st, [1, 2], 10, dbl.PipelineOptions(t_draft=0.0))
    r = dbl.run(d, t, st, [2, 2, 4], 1)  # max_new_tokens = 1 (test_pipeline.cpp:229-236)
    assert len(r.output) == 1


def test_formats_through_device_objects(dbl, tmp_path):
    """save_model / save_index / load_index (model.cpp:230-242, datastore.cpp:189-201) on device objects:
    the files equal the reference-written ones byte for byte."""
    d, t = _config1_models(dbl)
    p = tmp_path / "t.model-v1"
    dbl.save_model(t, str(p))
    assert p.read_text() == open(os.path.join(GOLDEN, "config1_target.model-v1")).read()
    t2 = dbl.load_model(str(p))
    assert dbl.forward_batch(t2, [2, 2, 4], [28, 2]) == dbl.forward_batch(t, [2, 2, 4], [28, 2])
    st = _config1_store(dbl)
    q = tmp_path / "prior.dstore-v1"
    dbl.save_index(st, str(q))
    assert q.read_text() == open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read()
    st2 = dbl.HierarchicalDatastore(3, 10)
    dbl.load_index(str(q), st2)
    assert st2.prior.sequences == st.prior.sequences
    assert st2.lookup([2, 4], 10).candidates == st.lookup([2, 4], 10).candidates
