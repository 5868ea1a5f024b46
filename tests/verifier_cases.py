"""Random verifier cases shared by the CPU (oracle vs reference) and GPU (device vs oracle) tests.
Distributions are ragged fp64 rows with exact zeros, ties and near-degenerate mass, like the
reference's ProbVectors; about a quarter of the cases hit the reference's error paths."""
import random


def _dist(rng: random.Random, v: int):
    w = [0.0 if rng.random() < 0.25 else rng.choice([rng.random(), 0.5, 1e-12]) for _ in range(v)]
    if rng.random() < 0.1:
        w = [0.0] * v  # degenerate row
    s = sum(w)
    return [x / s for x in w] if s > 0 else w


def cases(seed: int, n: int):
    rng = random.Random(seed)
    for _ in range(n):
        v = rng.randint(2, 24)
        nd = rng.randint(0, 6)
        draft = [rng.randrange(v) for _ in range(nd)]
        temp = rng.choice([0.0, 0.0, 0.7, 1.0])
        # the reference indexes draft_probs[k] unchecked when T > 0 (verification.cpp:73, :128): stay
        # inside its defined domain there; greedy cases may still leave rows uncovered (checked paths)
        fr = None if rng.random() < 0.3 else rng.randint(0, nd)
        nd_rows = max(nd, (fr or 0) + 1) if temp > 0 else rng.randint(max(0, nd - 1), nd + 1)
        dprobs = [_dist(rng, v) for _ in range(nd_rows)]
        ng = rng.randint(0, nd + 3)
        gtok = list(draft[:rng.randint(0, nd)]) + [rng.randrange(v) for _ in range(max(0, ng - nd))]
        gprobs = [_dist(rng, v) for _ in range(rng.randint(0, nd + 2))]
        tprobs = [_dist(rng, v) for _ in range(rng.randint(max(0, nd - 1), nd + 1))]
        yield dict(draft=draft, dprobs=dprobs, gtok=gtok, gprobs=gprobs, tprobs=tprobs, first_reject=fr,
                   temperature=temp, seed=rng.randrange(1 << 62), x=rng.randrange(v), v=v)
