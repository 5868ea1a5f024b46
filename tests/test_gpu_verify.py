"""GPU: the device verifier API (csrc/verify.cu via the C-ABI) against the oracle restatement on the
known-answer cases and the random cases of tests/verifier_cases.py — outcomes, every mt19937_64 draw
and exception types identical (the oracle is pinned to the reference in test_verifier.py)."""
import pytest

from verifier_cases import cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dbl():
    import paper_2601_05524_b200 as dbl
    assert dbl._capi.lib().dbl_device_ok() == 1
    return dbl


@pytest.fixture(scope="module")
def ov(oracle):
    from oracle.pyoracle import OracleVerifier
    return OracleVerifier(oracle)


def test_device_rng_matches_reference_stream(dbl, ov):
    for seed, rnd, lane in ((0, 0, 0), (11, 3, 2), (2**63 + 5, 97, 1)):
        d, o = dbl.derive_rng(seed, rnd, lane), ov.derive_rng(seed, rnd, lane)
        assert dbl_list(d.uniform(700)) == [ov.uniform(o) for _ in range(700)]
    d, o = dbl.Rng(42), ov.rng(42)
    assert d.uniform() == ov.uniform(o)


def dbl_list(a):
    return [float(x) for x in a]


def test_device_guided_output_known_answers(dbl):
    g = dbl.Rng(1)
    G = dbl.GuidanceChain
    o = dbl.guided_output([3, 4], [], G(tokens=[3, 4, 7, 8]), None, 0.0, g)
    assert (o.accepted_len, o.committed, o.kind) == (2, [3, 4, 7, 8], "extension")
    o = dbl.guided_output([3, 4, 5], [], G(tokens=[3, 6, 7]), 1, 0.0, g)
    assert (o.accepted_len, o.committed, o.kind) == (1, [3, 6, 7], "correction")
    o = dbl.guided_output([3, 4], [], G(tokens=[3], probs=[[0.9, 0.1], [0.1, 0.9]]), 1, 0.0, g)
    assert o.committed == [3, 1]
    with pytest.raises(dbl.InvalidArgument):
        dbl.guided_output([3, 4], [], G(), 1, 0.0, g)
    o = dbl.guided_output([0, 1], [[0.9, 0.1], [0.2, 0.5, 0.3]],
                          G(tokens=[0, 2, 4], probs=[[0.9, 0.1], [0.6, 0.1, 0.3]]), 1, 1.0, dbl.Rng(8))
    assert (o.accepted_len, o.committed, o.kind) == (1, [0, 0], "residual_correction")


def _outcome(f):
    try:
        return ("ok", f())
    except Exception as e:  # noqa: BLE001
        name = type(e).__name__
        return ("err", {"OracleInvalidArgument": "InvalidArgument", "OracleRuntimeError": "DoubleError",
                        "InvalidArgument": "InvalidArgument", "DoubleError": "DoubleError"}.get(name, name))


def test_device_verifier_matches_oracle(dbl, ov):
    for c in cases(seed=2024, n=300):
        d, o = dbl.Rng(c["seed"]), ov.rng(c["seed"])
        G = dbl.GuidanceChain(tokens=c["gtok"], probs=c["gprobs"])

        def dev_guided():
            r = dbl.guided_output(c["draft"], c["dprobs"], G, c["first_reject"], c["temperature"], d)
            return (r.accepted_len, r.committed, r.kind)

        a = _outcome(dev_guided)
        b = _outcome(lambda: ov.guided_output(c["draft"], c["dprobs"], c["gtok"], c["gprobs"], c["first_reject"],
                                              c["temperature"], o))
        assert a == b, (c, a, b)
        a = _outcome(lambda: dbl.verify_against_target(c["draft"], c["dprobs"], c["tprobs"], c["temperature"], d))
        b = _outcome(lambda: ov.verify_against_target(c["draft"], c["dprobs"], c["tprobs"], c["temperature"], o))
        assert a == b, (c, a, b)
        if c["tprobs"] and c["dprobs"]:
            p, q = c["tprobs"][0], c["dprobs"][0]
            assert _outcome(lambda: dbl.accept_prob(p, q, c["x"])) == _outcome(lambda: ov.accept_prob(p, q, c["x"]))
            assert _outcome(lambda: dbl.residual_sample(p, q, d)) == _outcome(lambda: ov.residual_sample(p, q, o))
            assert (_outcome(lambda: dbl.residual_sample_point_mass(p, c["x"], d)) ==
                    _outcome(lambda: ov.residual_sample_point_mass(p, c["x"], o)))
        assert d.uniform() == ov.uniform(o)
