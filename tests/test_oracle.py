"""CPU: the oracle restatement (oracle/specpar_oracle.c) pinned against the reference's golden
vectors (tests/golden/, produced by the unmodified reference) and, where oracle/_ref is built,
against the live reference on fresh random cases."""
import hashlib
import json
import os
import random

import pytest

from conftest import GOLDEN

CFG1 = json.load(open(os.path.join(GOLDEN, "config1.json")))


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def cfg_text(d):
    return "".join(f"{k}={v}\n" for k, v in d.items())


@pytest.mark.parametrize("method", list(CFG1["methods"]))
def test_config1_all_methods_bit_exact(oracle, method):
    out, js, met = oracle.run_config(CFG1["config"], method)
    want = CFG1["methods"][method]
    assert out == want["output"]
    assert sha(js) == want["jsonl_sha256"]
    assert met == list(want["metrics"].values())


def test_config1_appendix_b_anchors(oracle):
    # greedy output sha, double/psd/vanilla trace shas, double metrics
    out, js, met = oracle.run_config(CFG1["config"], "double")
    assert hashlib.sha256(("".join(f"{t} " for t in out) + "\n").encode()).hexdigest() == \
        "d911443cd7df7737f38ce90268f1e9105d6eb01facf70a8fb4caee9063d94305"
    assert sha(js) == "7587b2f768e7e815be523b31a26e35bd9e268f2e4532ad9b9713ec976bf3de76"
    assert met[:6] == [260, 86, 107.5, 4.0, pytest.approx(1.10078, abs=1e-5), pytest.approx(2.4186, abs=1e-4)]
    assert js.splitlines()[0] == ('{"round":0,"mode":"pre_verify","pending":0,"draft_len":6,'
                                  '"draft_matched":[4,0],"target_matched":2,"target_source":"prior",'
                                  '"accepted_pending":0,"pending_reject":false,"rejected":true,'
                                  '"committed":3,"kind":"extend_drop_draft","clock_delta":1.25}')


def test_config1_setup_serialisations(oracle):
    corpus = oracle.gen_corpus(32, 0.95, 4096, 11)
    assert corpus[0][:8] == CFG1["prompt"]
    for order, key in ((1, "draft_model_v1"), (2, "target_model_v1")):
        assert sha(oracle.table_build(corpus, order, 0.1, 32).serialize()) == CFG1["sha256"][key]
    st = oracle.store(3, 10)
    for i, s in enumerate(corpus[:10]):
        st.insert(0, s, i)
    assert sha(st.serialize(0)) == CFG1["sha256"]["prior_dstore_v1"]
    # model-v1 parse round trip
    text = open(os.path.join(GOLDEN, "config1_target.model-v1")).read()
    assert oracle.table_parse(text).serialize() == text


def test_acceptance_set_100_configs(oracle):
    acc = json.load(open(os.path.join(GOLDEN, "acceptance100.json")))
    assert len(acc) == 100
    for case in acc:
        t = cfg_text(case["config"])
        out, js, met = oracle.run_config(t, "double")
        assert sha(" ".join(map(str, out))) == case["output_sha256"]
        assert sha(js) == case["jsonl_sha256"]
        assert met == list(case["metrics"].values())
        # lossless: Double == target-only greedy AR (acceptance.cpp:99-125)
        ar, _, _ = oracle.run_config(t, "vanilla_ar")
        assert sha(" ".join(map(str, ar))) == case["ar_output_sha256"] == case["output_sha256"]


def _replay_lookups(oracle, case):
    st = oracle.store(case["max_order"], 10)
    st.set_rejected_enabled(case["rejected_enabled"])
    for layer, toks, step in case["inserts"]:
        st.insert(layer, toks, step)
    got = [list(st.lookup(ctx, d)) for ctx, d in case["queries"]]
    return got, st.stats()


def test_lookup_golden_fuzz(oracle):
    cases = json.load(open(os.path.join(GOLDEN, "lookups.json")))
    for case in cases:
        got, stats = _replay_lookups(oracle, case)
        assert got == case["results"]
        assert stats == case["stats"]


def test_lookup_known_answers(oracle):
    # test_datastore.cpp:62-159 restated
    st = oracle.store(3, 10)
    st.insert(0, [1, 2, 3, 4, 5, 6], 0)
    assert st.lookup([9, 2, 3], 10) == ([4, 5, 6], "prior", 2)
    st = oracle.store(3, 10)
    st.insert(0, [1, 2, 3, 4, 5, 6, 7, 8], 0)
    assert st.lookup([1, 2], 3)[0] == [3, 4, 5]
    assert st.lookup([1, 2], 100)[0] == [3, 4, 5, 6, 7, 8]
    st = oracle.store(3, 10)
    st.insert(0, [2, 3, 9], 0)
    st.insert(1, [1, 2, 3, 7], 1)
    assert st.lookup([1, 2, 3], 10) == ([7], "dynamic", 3)
    st = oracle.store(2, 10)
    st.insert(0, [1, 2, 5], 0); st.insert(1, [1, 2, 6], 1); st.insert(2, [1, 2, 7], 2)
    assert st.lookup([1, 2], 10)[:2] == ([5], "prior")
    st = oracle.store(2, 10)
    st.insert(2, [1, 2, 7, 8], 0)
    assert st.lookup([1, 2], 10)[:2] == ([7, 8], "rejected")
    st.set_rejected_enabled(False)
    assert st.lookup([1, 2], 10)[1] == "miss"
    st = oracle.store(2, 10)
    st.insert(1, [1, 2, 5], 0); st.insert(1, [1, 2, 6], 3); st.insert(1, [1, 2, 4], 1)
    assert st.lookup([1, 2], 10)[0] == [6]
    st = oracle.store(3, 10)
    assert st.lookup([1, 2, 9, 1, 2, 8, 1, 2], 10) == ([8, 1, 2], "context", 2)
    assert st.lookup([5, 1, 2, 3, 7, 1, 2, 3], 2) == ([7, 1], "context", 3)
    assert st.lookup([1, 2, 3], 10) == ([], "miss", 0)
    st = oracle.store(2, 10)
    st.insert(0, [1, 2, 5], 0)
    st.lookup([1, 2], 10); st.lookup([1, 2], 10); st.lookup([7, 8], 10)
    assert st.stats() == [3, 2, 0, 0, 0, 1]


def test_lookup_live_reference_fuzz(oracle, reference):
    rng = random.Random(7)
    for _ in range(200):
        mo = rng.choice([1, 2, 3, 4])
        vocab = rng.choice([2, 3, 5, 9])
        inserts = [(rng.choice([0, 1, 2]), [rng.randrange(vocab) for _ in range(rng.randint(1, 30))],
                    rng.randint(0, 6)) for _ in range(rng.randint(0, 10))]
        queries = [([rng.randrange(vocab) for _ in range(rng.randint(1, 20))], rng.randint(1, 12))
                   for _ in range(8)]
        rej = rng.random() < 0.7
        want, wstats = reference.lookup_batch(mo, inserts, queries, rejected_enabled=rej)
        got, stats = _replay_lookups(oracle, {"max_order": mo, "rejected_enabled": rej,
                                              "inserts": inserts, "queries": queries})
        assert got == [list(x) for x in want]
        assert stats == wstats


def test_live_reference_random_configs(oracle, reference):
    rng = random.Random(11)
    for i in range(25):
        d = dict(vocab=rng.choice([8, 16, 40]), rho=rng.choice([0.0, 0.3, 0.9, 1.0]),
                 corpus_len=rng.choice([512, 2048]), draft_order=rng.choice([1, 2, 3]),
                 target_order=rng.choice([1, 2, 3]), t_draft=rng.choice([0.2, 0.3, 0.5]),
                 t_lookup=rng.choice([0.0, 0.05]), t_sync=rng.choice([0.0, 0.01]),
                 gamma=rng.choice([0, 1, 3, 6]), depth=rng.choice([1, 3, 10, 16]),
                 ngram=rng.choice([1, 2, 3, 4]), prior_rounds=rng.choice([0, 3, 10]),
                 seed=500 + i, max_new_tokens=rng.choice([1, 17, 128]),
                 prompt_len=rng.choice([1, 8, 30]), rejected_cache=rng.choice([0, 1]))
        t = cfg_text(d)
        for m in ("double", "psd", "target_retrieval", "draft_retrieval", "sd", "vanilla_ar"):
            assert oracle.run_config(t, m) == reference.run_config(t, m), (d, m)


def test_callback_loop_matches_reference(oracle, reference):
    """orc_run with callback models == the reference run() through the --wrap seam."""
    from oracle.pyoracle import make_argmax_callback
    rng = random.Random(3)
    V = 23
    tw = [[rng.random() for _ in range(V)] for _ in range(V * V)]
    dw = [[rng.random() for _ in range(V)] for _ in range(V)]

    def tgt(ctx, cands):
        c = ctx + cands
        return [max(range(V), key=lambda v: (tw[(c[i - 2] if i >= 2 else 0) * V + c[i - 1]][v], -v))
                for i in range(len(ctx), len(c) + 1)]

    def dft(ctx, cands):
        c = ctx + cands
        return [max(range(V), key=lambda v: (dw[c[i - 1]][v], -v)) for i in range(len(ctx), len(c) + 1)]
    tcb, dcb = make_argmax_callback(tgt), make_argmax_callback(dft)
    prior = [[rng.randrange(1, V) for _ in range(40)] for _ in range(4)]
    prompt = [rng.randrange(1, V) for _ in range(12)]
    for gamma, depth in ((1, 3), (3, 10), (5, 4)):
        want = reference.run_callback(V, dcb, tcb, prior, prompt, 60, gamma=gamma, depth=depth)
        st = oracle.store(3, depth)
        for i, s in enumerate(prior):
            st.insert(0, s, i)
        got = oracle.run(V, dcb, V, tcb, st, prompt, 60, gamma=gamma, depth=depth)
        assert got == want
