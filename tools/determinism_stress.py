"""Stress one forward shape: N identical forward_logits calls -> number of distinct results.
    python tools/determinism_stress.py model ctx rows reps"""
import hashlib
import os
import random
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402

name, ctx_len, nrows, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = dbl.transformer_config(name, seed=7, max_seq=1408, n_layers=2)
m = dbl.Transformer(cfg)
rng = random.Random(5)
ctx = [rng.randrange(cfg.vocab) for _ in range(ctx_len)]
cands = [rng.randrange(cfg.vocab) for _ in range(nrows - 1)]
hs, first = {}, {}
for _ in range(reps):
    lg = dbl.forward_logits(m, ctx, cands)
    h = hashlib.sha256(np.ascontiguousarray(lg).tobytes()).hexdigest()[:10]
    hs[h] = hs.get(h, 0) + 1
    first.setdefault(h, lg)
if len(first) > 1:
    ks = sorted(first, key=lambda k: -hs[k])
    a = first[ks[0]]
    for k in ks[1:]:
        d = np.abs(first[k] - a)
        rows = np.nonzero(d.max(axis=1) > 0)[0].tolist()
        print(f"  variant {k} x{hs[k]}: rows differing {rows}, max|diff| {d.max():.3e} (max|logit| {np.abs(a).max():.3e}), "
              f"cols differing per row {[int((d[r] > 0).sum()) for r in rows][:12]}", flush=True)
print(f"{os.path.basename(os.environ.get('DBL_LIB', 'current'))} smem={os.environ.get('DBL_FWD_SMEM_KB', '-')} {name} ctx={ctx_len} rows={nrows}: "
      f"{len(hs)} distinct in {reps} {sorted(hs.values(), reverse=True)}", flush=True)
