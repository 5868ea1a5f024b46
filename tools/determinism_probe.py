"""Repeat identical forwards and count distinct results (the forward must be bitwise deterministic:
the lossless DOUBLE == AR identity depends on it).  python tools/determinism_probe.py [model] [reps]"""
import hashlib
import os
import random
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-0.6b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = dbl.transformer_config(name, seed=7, max_seq=1408, n_layers=2)
m = dbl.Transformer(cfg)
rng = random.Random(5)
for ctx_len, nrows in ((288, 1), (1152, 1), (288, 12), (1152, 12), (288, 40)):
    ctx = [rng.randrange(cfg.vocab) for _ in range(ctx_len)]
    cands = [rng.randrange(cfg.vocab) for _ in range(nrows - 1)]
    hs, args = set(), set()
    for _ in range(reps):
        lg = dbl.forward_logits(m, ctx, cands)
        hs.add(hashlib.sha256(np.ascontiguousarray(lg).tobytes()).hexdigest()[:12])
        args.add(tuple(dbl.forward_batch(m, ctx, cands)))
    print(f"{name} ctx={ctx_len} rows={nrows}: {len(hs)} distinct logits, {len(args)} distinct argmax rows"
          + ("" if len(hs) == 1 and len(args) == 1 else "  <-- NONDETERMINISTIC"), flush=True)
