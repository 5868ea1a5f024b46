"""GPU: the rest of the reference's decode-path API through the C-ABI — run_round /
rollback / PipelineState, the drafter (accept_with_model / retrieval_forward / iterative_draft /
measure_amt), the model helpers (tempered / argmax_token / sample), compute_metrics / traces_to_jsonl /
write_traces, store copies and the bulk build_prior.  The round-at-a-time loop must reproduce run()
(and so the reference's golden JSONL) exactly; the helpers must reproduce the reference's semantics."""
import hashlib
import json
import os
import random

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CFG1 = json.load(open(os.path.join(GOLDEN, "config1.json")))


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1
    return dbl


def _config1(dbl):
    from paper_2601_05524_b200.specpar import parse_dstore_v1
    d = dbl.TableModel.from_model_v1(open(os.path.join(GOLDEN, "config1_draft.model-v1")).read())
    t = dbl.TableModel.from_model_v1(open(os.path.join(GOLDEN, "config1_target.model-v1")).read())
    _, seqs = parse_dstore_v1(open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read())
    return d, t, seqs


def drive_rounds(dbl, draft, target, store, prompt, max_new, opts, eos):
    """run() (pipeline.cpp:264-323) restated over run_round, exactly as the reference's loop."""
    st = dbl.PipelineState(committed=list(prompt), prev_tokens=opts.gamma, last_committed_len=len(prompt))
    store.record_accepted(prompt)
    traces = []
    scanned, done = len(prompt), False
    while not done:
        traces.append(dbl.run_round(st, draft, target, store, opts))
        while scanned < len(st.committed):
            if st.committed[scanned] == eos:
                st.committed = st.committed[:scanned + 1]
                done = True
                break
            scanned += 1
        if len(st.committed) - len(prompt) >= max_new:
            done = True
    return st, traces


def test_run_round_loop_reproduces_config1_golden(dbl):
    d, t, seqs = _config1(dbl)
    want = CFG1["methods"]["double"]
    st0 = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st0, seqs, len(seqs))
    opts = dbl.PipelineOptions(gamma=2, depth=10, t_target=1.0, t_draft=0.625)
    st, traces = drive_rounds(dbl, d, t, st0, CFG1["prompt"], 256, opts, t.vocab_size - 1)
    assert st.committed[len(CFG1["prompt"]):][:256] == want["output"]
    assert sha(dbl.traces_to_jsonl(traces)) == want["jsonl_sha256"]
    m = dbl.compute_metrics(traces, 1.0)
    assert [m["tokens"], m["rounds"], m["clock"], m["m"], m["amt"], m["speedup"]] == \
        [want["metrics"][k] for k in ("tokens", "rounds", "clock", "m", "amt", "speedup")]
    assert abs(st.clock - want["metrics"]["clock"]) < 1e-9


@pytest.mark.parametrize("temperature", [0.0, 1.0, 0.7])
def test_run_round_loop_equals_run_on_transformers(dbl, temperature):
    """The session keeps the lanes' KV between rounds; a round-at-a-time decode == run() bitwise."""
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=31, max_seq=1024))
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=32, max_seq=1024))
    rng = random.Random(4)
    prompt = [rng.randrange(1, 900) for _ in range(40)]
    prior = [[rng.randrange(1, 900) for _ in range(30)] for _ in range(6)] + [prompt[5:35]]
    opts = dbl.PipelineOptions(gamma=3, depth=10, temperature=temperature, rng_seed=9)
    s1, s2 = dbl.HierarchicalDatastore(3, 10), dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(s1, prior, 10)
    dbl.build_prior(s2, prior, 10)
    r = dbl.run(drf, tgt, s1, prompt, 48, opts)
    st, traces = drive_rounds(dbl, drf, tgt, s2, prompt, 48, opts, tgt.vocab_size - 1)
    assert st.committed[len(prompt):][:48] == r.output
    assert dbl.traces_to_jsonl(traces) == r.jsonl


def test_rollback_and_fresh_state_equivalence_on_transformers(dbl):
    """test_pipeline.cpp:151-197 on transformer models: rollback semantics and 'rollback to the
    committed boundary equals never having speculated' with copied stores."""
    tgt = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=41, max_seq=1024))
    drf = dbl.Transformer(dbl.transformer_config("tiny-qwen-draft", seed=42, max_seq=1024))
    st = dbl.PipelineState(committed=[1, 2, 3, 4, 5], speculative=[6, 7], spec_probs=[None, None],
                           mode="post_verify", last_committed_len=3)
    dbl.rollback(st, 4)
    assert st.committed == [1, 2, 3, 4] and st.speculative == [] and st.mode == "pre_verify"
    dbl.rollback(st, 4)
    assert st.committed == [1, 2, 3, 4]
    with pytest.raises(dbl.InvalidArgument):
        dbl.rollback(st, 99)
    with pytest.raises(dbl.LogicError):
        dbl.rollback(st, 2)
    prompt = list(range(3, 40))
    base = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(base, [prompt[2:30], prompt[10:]], 10)
    opts = dbl.PipelineOptions(gamma=4)
    a = dbl.PipelineState(committed=list(prompt), prev_tokens=4, last_committed_len=len(prompt))
    store_a = base.copy()
    dbl.run_round(a, drf, tgt, store_a, opts)
    after = list(a.committed)
    dbl.rollback(a, len(a.committed))
    a.prev_tokens = 4
    b = dbl.PipelineState(committed=after, prev_tokens=4, round=a.round, last_committed_len=len(after))
    store_b, store_a2 = store_a.copy(), store_a.copy()
    ta = dbl.run_round(a, drf, tgt, store_a2, opts)
    tb = dbl.run_round(b, drf, tgt, store_b, opts)
    assert a.committed == b.committed and a.speculative == b.speculative and ta == tb
    assert store_a2.dynamic.sequences == store_b.dynamic.sequences
    # inconsistent state -> logic_error (test_pipeline.cpp:138-149)
    bad = dbl.PipelineState(committed=list(prompt), speculative=[1, 2], spec_probs=[None, None],
                            mode="post_verify", prev_tokens=3)
    with pytest.raises(dbl.LogicError):
        dbl.run_round(bad, drf, tgt, base, opts)


def test_store_copy_is_deep_and_bulk_prior_equals_inserts(dbl, oracle):
    rng = random.Random(7)
    seqs = [[rng.randrange(0, 50) for _ in range(rng.randrange(1, 40))] for _ in range(200)]
    bulk = dbl.HierarchicalDatastore(3, 10)
    bulk.prior = dbl.build_prior(seqs, 3, 150)  # the reference's signature: an NGramIndex value
    one = dbl.HierarchicalDatastore(3, 10)
    for i, q in enumerate(seqs[:150]):
        one.prior.insert(q, i)
    assert bulk.prior.sequences == one.prior.sequences
    assert bulk.prior.occurrence_count() == one.prior.occurrence_count() == \
        dbl.build_prior(seqs, 3, 150).occurrence_count()
    cp = bulk.copy()
    queries = [[rng.randrange(0, 50) for _ in range(rng.randrange(1, 8))] for _ in range(300)]
    for q in queries:
        a, b, c = bulk.lookup(q, 10), one.lookup(q, 10), cp.lookup(q, 10)
        assert (a.candidates, a.source, a.matched_order) == (b.candidates, b.source, b.matched_order) == \
            (c.candidates, c.source, c.matched_order)
    cp.dynamic.insert([1, 2, 3, 4], 999)
    assert bulk.dynamic.sequences == [] and cp.dynamic.sequences == [[1, 2, 3, 4]]
    with pytest.raises(dbl.InvalidArgument):
        dbl.build_prior(seqs, 3, -1)


def test_model_helpers(dbl):
    rng = np.random.default_rng(3)
    for V in (2, 5, 1000, 151936):
        rows = [rng.random(V) for _ in range(4)]
        rows[1][V // 3] = rows[1][V - 1] = 2.0  # a tie: the lowest id
        rows[2][:] = 0.25
        assert dbl.argmax_rows(rows) == [int(np.argmax(r)) for r in rows]
        assert dbl.argmax_token(rows[0]) == int(np.argmax(rows[0]))
    with pytest.raises(dbl.DoubleError):
        dbl.argmax_token([0.0, 0.0, 0.0])
    p = np.array([0.1, 0.2, 0.3, 0.4])
    assert dbl.tempered(p, 1.0).tolist() == p.tolist()
    sharp = dbl.tempered(p, 0.25)
    assert abs(sharp[2] - 0.3 ** 4 / np.sum(p ** 4)) < 1e-12
    a, b = dbl.Rng(7), dbl.Rng(7)
    assert dbl.sample([0.1, 0.7, 0.2], 0.0, a) == 1 and a.uniform() == b.uniform()
    c, e = dbl.Rng(7), dbl.Rng(7)
    e.uniform()
    dbl.sample([0.1, 0.7, 0.2], 1.0, c)
    assert c.uniform() == e.uniform()


def test_drafter_known_answers(dbl):
    """test_speculation.cpp:39-200 (greedy cases) through the device drafter."""
    dists = [[0.0, 1.0, 0.0], [0.0, 0.0, 1.0], [1.0, 0.0, 0.0]]
    r = dbl.accept_with_model(dists, [1, 2])
    assert (r.matched_len, r.emitted, len(r.probs)) == (2, [1, 2, 0], 3)
    r = dbl.accept_with_model(dists, [1, 0])
    assert (r.matched_len, r.emitted, len(r.probs)) == (1, [1, 2], 2) and r.probs[1].tolist() == dists[1]
    assert dbl.accept_with_model([dists[0]], []).emitted == [1]
    with pytest.raises(dbl.InvalidArgument):
        dbl.accept_with_model(dists, [1, 2, 0])
    r = dbl.accept_with_model(dists, [7, 2])
    assert (r.matched_len, r.emitted) == (0, [1])
    V = 5
    nxt = [1, 2, 3, 4, 1]
    probs = [1.0 if t == nxt[a] else 0.0 for a in range(V) for t in range(V)]
    m = dbl.TableModel(1, V, list(range(V)), probs, [0.2] * V)
    st = dbl.HierarchicalDatastore(3, 10)
    st.prior.insert([1, 2, 3, 4], 0)
    r = dbl.retrieval_forward(m, st, [1, 2], 10)
    assert (r.source, r.matched_len, r.emitted) == ("prior", 2, [3, 4, 1])
    r = dbl.retrieval_forward(m, dbl.HierarchicalDatastore(3, 10), [3], 10)
    assert (r.source, r.matched_len, r.emitted, len(r.probs)) == ("miss", 0, [4], 1)
    before = st.stats.lookups
    r = dbl.retrieval_forward(m, st, [1, 2], 10, use_retrieval=False)
    assert (r.matched_len, r.emitted) == (0, [3]) and st.stats.lookups == before
    st2 = dbl.HierarchicalDatastore(3, 10)
    st2.prior.insert([1, 2, 3, 4, 1, 2, 3, 4], 0)
    ch = dbl.iterative_draft(m, st2, [1], 3, 4)
    grown, flat = [1], []
    for j in range(3):
        seg = dbl.retrieval_forward(m, st2, grown, 4)
        grown += seg.emitted
        flat += seg.emitted
        assert seg.emitted == ch.segments[j].emitted
    assert ch.tokens == flat and ch.total_len == len(flat) and len(ch.probs) == len(flat)
    with pytest.raises(dbl.InvalidArgument):
        dbl.iterative_draft(m, st2, [1], 0, 4)
    assert dbl.measure_amt([2, 0, 7]) == 3.0
    with pytest.raises(dbl.InvalidArgument):
        dbl.measure_amt([])


def test_drafter_on_transformer_matches_decode_loop_semantics(dbl):
    """retrieval_forward on a transformer == lookup + forward_batch argmax walk (greedy), and the
    sampled accept consumes the reference's draws (T = 1: same emitted stream from the same seed)."""
    m = dbl.Transformer(dbl.transformer_config("tiny-qwen", seed=51, max_seq=512))
    rng = random.Random(5)
    ctx = [rng.randrange(1, 1000) for _ in range(30)]
    st = dbl.HierarchicalDatastore(3, 10)
    st.prior.insert(ctx[10:25] + [rng.randrange(1, 1000) for _ in range(12)], 0)
    q = ctx[:24]
    hit = st.lookup(q, 10)
    assert hit.source == "prior" and len(hit.candidates) == 10
    am = dbl.forward_batch(m, q, hit.candidates)
    s = 0
    while s < len(hit.candidates) and hit.candidates[s] == am[s]:
        s += 1
    r = dbl.retrieval_forward(m, st, q, 10)
    assert r.matched_len == s and r.emitted == hit.candidates[:s] + [am[s]] and r.source == "prior"
    assert len(r.probs) == s + 1 and int(np.argmax(r.probs[-1])) == am[s]
    a = dbl.retrieval_forward(m, st, q, 10, temperature=1.0, rng=dbl.Rng(3))
    b = dbl.retrieval_forward(m, st, q, 10, temperature=1.0, rng=dbl.Rng(3))
    assert a.emitted == b.emitted


def test_write_traces(dbl, tmp_path):
    traces = [{"round": 0, "mode": "pre_verify", "committed": 7, "clock_delta": 1.0, "kind": "extend_drop_draft",
               "target_source": "prior", "draft_matched": [1, 0]},
              {"round": 1, "mode": "post_verify", "pending_reject": True, "rejected": True, "accepted_pending": 0,
               "committed": 1, "clock_delta": 1.0, "kind": "pending_reject", "target_source": "miss"}]
    m = dbl.compute_metrics(traces)
    assert m["m"] == 4.0 and m["tokens"] == 8
    p = tmp_path / "t.jsonl"
    dbl.write_traces(traces, str(p))
    assert p.read_text() == dbl.traces_to_jsonl(traces)
    assert [json.loads(x)["kind"] for x in p.read_text().splitlines()] == ["extend_drop_draft", "pending_reject"]
    with pytest.raises(dbl.InvalidArgument):
        dbl.compute_metrics([])
