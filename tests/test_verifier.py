"""Verifier API (verification.hpp:30-53) and RNG (rng.hpp): the oracle restatement against the
reference's own known-answer tests (test_verification.cpp:174-245) and against the unmodified
reference (oracle/_ref) on random cases — every outcome, draw and exception type identical."""
import pytest

from verifier_cases import cases


@pytest.fixture(scope="module")
def ov(oracle):
    from oracle.pyoracle import OracleVerifier
    return OracleVerifier(oracle)


@pytest.fixture(scope="module")
def rv(reference):
    from oracle.pyoracle import ReferenceVerifier
    return ReferenceVerifier(reference)


def test_guided_output_known_answers(ov):
    from oracle.pyoracle import OracleInvalidArgument
    g = ov.rng(1)
    # test_verification.cpp:174-185 all accepted
    assert ov.guided_output([3, 4], [], [3, 4], [], None, 0.0, g) == (2, [3, 4], "all_accepted")
    # :187-202 extension needs a covering guidance prefix
    assert ov.guided_output([3, 4], [], [3, 4, 7, 8], [], None, 0.0, g) == (2, [3, 4, 7, 8], "extension")
    assert ov.guided_output([3, 4], [], [3, 9, 7, 8], [], None, 0.0, g) == (2, [3, 4], "all_accepted")
    # :204-214 greedy rejection keeps the guidance tail
    assert ov.guided_output([3, 4, 5], [], [3, 6, 7], [], 1, 0.0, g) == (1, [3, 6, 7], "correction")
    # :216-229 rejection past the chain falls back to argmax; uncovered -> invalid_argument
    assert ov.guided_output([3, 4], [], [3], [[0.9, 0.1], [0.1, 0.9]], 1, 0.0, g) == (1, [3, 1], "correction")
    with pytest.raises(OracleInvalidArgument):
        ov.guided_output([3, 4], [], [], [], 1, 0.0, g)
    # :231-245 stochastic rejection draws a residual (mass only on token 0) and drops the tail
    acc, out, kind = ov.guided_output([0, 1], [[0.9, 0.1], [0.2, 0.5, 0.3]], [0, 2, 4],
                                      [[0.9, 0.1], [0.6, 0.1, 0.3]], 1, 1.0, ov.rng(8))
    assert (acc, out, kind) == (1, [0, 0], "residual_correction")


def _same(fa, fb):
    """both return the same value, or both raise the same exception class"""
    try:
        a = ("ok", fa())
    except Exception as e:  # noqa: BLE001
        a = ("err", type(e).__name__)
    try:
        b = ("ok", fb())
    except Exception as e:  # noqa: BLE001
        b = ("err", type(e).__name__)
    assert a == b, (a, b)
    return a


def test_rng_streams_match_reference(ov, rv):
    for seed, rnd, lane in ((0, 0, 0), (11, 3, 2), (2**63 + 5, 97, 1)):
        go, gr = ov.derive_rng(seed, rnd, lane), rv.derive_rng(seed, rnd, lane)
        assert [ov.uniform(go) for _ in range(700)] == [rv.uniform(gr) for _ in range(700)]
        go, gr = ov.rng(seed), rv.rng(seed)
        assert [ov.uniform(go) for _ in range(5)] == [rv.uniform(gr) for _ in range(5)]


def test_verifier_matches_reference_on_random_cases(ov, rv):
    kinds = set()
    for c in cases(seed=2024, n=1500):
        go, gr = ov.rng(c["seed"]), rv.rng(c["seed"])
        r = _same(lambda: ov.guided_output(c["draft"], c["dprobs"], c["gtok"], c["gprobs"], c["first_reject"],
                                           c["temperature"], go),
                  lambda: rv.guided_output(c["draft"], c["dprobs"], c["gtok"], c["gprobs"], c["first_reject"],
                                           c["temperature"], gr))
        kinds.add(r[1][2] if r[0] == "ok" else r[1])
        _same(lambda: ov.verify_against_target(c["draft"], c["dprobs"], c["tprobs"], c["temperature"], go),
              lambda: rv.verify_against_target(c["draft"], c["dprobs"], c["tprobs"], c["temperature"], gr))
        if c["tprobs"] and c["dprobs"]:
            p, q = c["tprobs"][0], c["dprobs"][0]
            _same(lambda: ov.accept_prob(p, q, c["x"]), lambda: rv.accept_prob(p, q, c["x"]))
            _same(lambda: ov.residual_sample(p, q, go), lambda: rv.residual_sample(p, q, gr))
            _same(lambda: ov.residual_sample_point_mass(p, c["x"], go),
                  lambda: rv.residual_sample_point_mass(p, c["x"], gr))
        assert ov.uniform(go) == rv.uniform(gr)  # the streams advanced identically
    assert {"all_accepted", "correction", "extension", "residual_correction"} <= kinds
