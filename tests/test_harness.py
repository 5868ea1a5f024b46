"""CPU: the harness in front of the device loop (harness.py) — config parsing, the synthetic corpus and
the table models are identical to the reference's (oracle/_ref, unmodified sources) and to the oracle."""
import json
import os
import random

import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def hz():
    from paper_2601_05524_b200 import harness
    return harness


def test_gen_corpus_matches_reference(hz, reference, oracle):
    rng = random.Random(9)
    for _ in range(8):
        vocab, rho, n, seed = rng.choice([8, 32, 1000]), rng.choice([0.0, 0.5, 0.95, 1.0]), rng.randint(5, 3000), rng.randrange(1 << 40)
        want = reference.gen_corpus(vocab, rho, n, seed)
        assert hz.gen_corpus(vocab, rho, n, seed) == want
        assert oracle.gen_corpus(vocab, rho, n, seed) == want


def test_table_model_matches_c_serializer(hz, oracle):
    from paper_2601_05524_b200.specpar import serialize_model
    for vocab, order, sm, seed in ((32, 1, 0.1, 11), (32, 2, 0.1, 11), (16, 3, 0.0, 4), (64, 2, 0.37, 7)):
        corpus = hz.gen_corpus(vocab, 0.9, 2048, seed)
        spec = hz.build_model_from_corpus(corpus, order, sm, vocab)
        text = serialize_model(spec.order, spec.vocab, spec.windows, spec.probs, spec.fallback, sm)
        assert text == oracle.table_build(corpus, order, sm, vocab).serialize()


def test_config1_setup_equals_reference_export(hz):
    c1 = json.load(open(os.path.join(GOLDEN, "config1.json")))
    from paper_2601_05524_b200.specpar import serialize_model, serialize_index
    cfg = hz.parse_config(c1["config"])
    assert (cfg.vocab, cfg.rho, cfg.gamma, cfg.effective_gamma(), cfg.method, cfg.engine) == (32, 0.95, 0, 2, "double", "serial")
    s = hz.build_setup(cfg)
    assert s.prompt == c1["prompt"]
    for spec, name in ((s.draft, "config1_draft.model-v1"), (s.target, "config1_target.model-v1")):
        text = serialize_model(spec.order, spec.vocab, spec.windows, spec.probs, spec.fallback, spec.smoothing)
        assert text == open(os.path.join(GOLDEN, name)).read()
    assert serialize_index(cfg.ngram, s.corpus[:cfg.prior_rounds]) == open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read()


def test_parse_config_errors_and_defaults(hz):
    cfg = hz.parse_config("# only comments\n\n  \n")
    assert cfg == hz.ExperimentConfig()
    for bad in ("vocab=abc\n", "nosuchkey=1\n", "just words\n", "method=fast\n", "engine=async\n"):
        with pytest.raises(hz.DoubleError):
            hz.parse_config(bad)
    for invalid in ("vocab=3\n", "rho=1.5\n", "t_draft=0\n", "depth=0\n", "temperature=-1\n"):
        with pytest.raises(hz.InvalidArgument):
            hz.parse_config(invalid)
    cfg = hz.parse_config("t_target = 1\nt_draft=0.3 # ratio 3.33\ngamma=0\n")
    assert cfg.effective_gamma() == 4
    assert hz.parse_config(hz.serialize_config(cfg)) == cfg


def test_gen_corpus_and_build_prior_reproduce_reference_prior(hz):
    """gen_corpus (harness.cpp:151-186) + build_prior / save_index (datastore.cpp:149-169) reproduce
    the reference's config-1 prior file byte for byte."""
    from paper_2601_05524_b200.specpar import serialize_index
    corpus = hz.gen_corpus(32, 0.95, 4096, 11)
    text = serialize_index(3, corpus[:10])
    assert text == open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read()
