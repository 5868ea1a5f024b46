"""CPU: the on-disk formats — model-v1 (model.cpp:155-242) and dstore-v1
(datastore.cpp:161-201) writers and readers, byte-exact against files written by the unmodified
reference (tests/golden/config1_*) and against the oracle's C serializer on random tables."""
import os
import random

import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def sp():
    from paper_2601_05524_b200 import specpar
    return specpar


@pytest.mark.parametrize("name", ["config1_draft.model-v1", "config1_target.model-v1"])
def test_model_v1_round_trip_reference_files(sp, name):
    text = open(os.path.join(GOLDEN, name)).read()
    order, vocab, w, p, f = sp.parse_model_v1(text)
    assert sp.serialize_model(order, vocab, w, p, f, sp.parse_model_v1_smoothing(text)) == text


def test_dstore_v1_round_trip_reference_file(sp):
    text = open(os.path.join(GOLDEN, "config1_prior.dstore-v1")).read()
    mo, seqs = sp.parse_dstore_v1(text)
    assert sp.serialize_index(mo, seqs) == text


def test_model_v1_matches_c_serializer_on_random_tables(sp, oracle):
    rng = random.Random(3)
    for _ in range(6):
        vocab = rng.choice([3, 16, 50])
        order = rng.choice([1, 2, 3])
        smoothing = rng.choice([0.1, 0.0, 1e-3, 0.37])
        corpus = [[rng.randrange(vocab) for _ in range(rng.randint(2, 60))] for _ in range(rng.randint(1, 8))]
        text = oracle.table_build(corpus, order, smoothing, vocab).serialize()
        o, v, w, p, f = sp.parse_model_v1(text)
        assert sp.serialize_model(o, v, w, p, f, sp.parse_model_v1_smoothing(text)) == text
        # rows given in any order serialize in std::map (lexicographic window) order
        perm = list(range(len(w)))
        rng.shuffle(perm)
        assert sp.serialize_model(o, v, w[perm], p[perm], f, smoothing) == text


def test_dstore_v1_matches_c_serializer(sp, oracle):
    rng = random.Random(5)
    st = oracle.store(3, 10)
    seqs = [[rng.randrange(40) for _ in range(rng.randint(1, 30))] for _ in range(12)]
    for i, s in enumerate(seqs):
        st.insert(0, s, i)
    assert sp.serialize_index(3, seqs) == st.serialize(0)


def test_format_errors(sp):
    with pytest.raises(sp.DoubleError):
        sp.parse_model_v1("model-v2 3 1 0.1\nfallback : 0.3 0.3 0.4\n")
    with pytest.raises(sp.DoubleError):
        sp.parse_model_v1("model-v1 3 1 0.1\n0 : 0.5 0.5 0\n")  # missing fallback row
    with pytest.raises(sp.DoubleError):
        sp.parse_model_v1("model-v1 3 2 0.1\n0 : 0.5 0.5 0\nfallback : 0.3 0.3 0.4\n")  # window length
    with pytest.raises(sp.DoubleError):
        sp.parse_dstore_v1("dstore-v2 3 0\n")
    with pytest.raises(sp.DoubleError):
        sp.parse_dstore_v1("dstore-v1 3 2\n1 2 3\n")  # truncated
