"""Hash of forward logits over a fixed set of (model, context, rows) cases: run once per library build
(DBL_LIB=...) and diff the outputs to show two builds compute bitwise-identical forwards.

    DBL_LIB=a.so python tools/logits_hash.py > a.txt; DBL_LIB=b.so python tools/logits_hash.py > b.txt
"""
import hashlib
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2601_05524_b200 as dbl  # noqa: E402

for name in ("qwen3-14b", "qwen3-0.6b", "llama-3.1-8b"):
    cfg = dbl.transformer_config(name, seed=7, max_seq=1408, n_layers=2)
    m = dbl.Transformer(cfg)
    rng = random.Random(5)
    for ctx_len, rows in ((288, 1), (288, 2), (288, 12), (288, 25), (288, 64), (1152, 12), (1152, 64)):
        ctx = [rng.randrange(cfg.vocab) for _ in range(ctx_len)]
        cands = [rng.randrange(cfg.vocab) for _ in range(rows - 1)]
        got = np.ascontiguousarray(dbl.forward_logits(m, ctx, cands), dtype=np.float32)
        print(name, ctx_len, rows, hashlib.sha256(got.tobytes()).hexdigest()[:16], flush=True)
    del m
