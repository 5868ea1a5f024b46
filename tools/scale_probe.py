"""BASELINE configs 3-5 model shapes on ONE B200 (unsharded; TP needs more GPUs than gpurun gives):
verify-forward cost vs the HBM roofline, and a short DOUBLE vs target-only AR decode."""
import gc
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2601_05524_b200 as dbl  # noqa: E402
from paper_2601_05524_b200 import _capi  # noqa: E402

PEAK = 6549.1
pairs = [("llama-3.2-1b", "llama-3.1-8b", 160), ("qwen3-1.7b", "qwen3-32b", 160), ("llama-3.2-1b", "llama-3.3-70b", 1024)]
only = sys.argv[1:] or None
for dname, tname, plen in pairs:
    if only and tname not in only:
        continue
    tgt = dbl.Transformer(dbl.transformer_config(tname, seed=1, max_seq=plen + 320))
    drf = dbl.Transformer(dbl.transformer_config(dname, seed=2, max_seq=plen + 320))
    for rows in (1, 8):
        out = np.zeros(8)
        _capi.check(_capi.lib().dbl_profile_forward(tgt._h, plen + 128, rows, 5, out.ctypes.data_as(_capi.F64P)))
        gbs = out[2] / out[0] / 1e6
        print(f"{tname}: {rows}-row verify forward at ctx {plen + 128}: {out[0]:.3f} ms, {out[2] / 1e9:.2f} GB "
              f"algorithmic -> {gbs:.0f} GB/s = {gbs / PEAK:.3f} of peak", flush=True)
    prompt, prior = bench.workload(tgt.cfg.vocab, plen, 101)
    st = dbl.HierarchicalDatastore(3, 10)
    dbl.build_prior(st, prior, 10)
    r = dbl.run(drf, tgt, st, prompt, 64, dbl.PipelineOptions(gamma=1, depth=10), want_jsonl=False)
    a = dbl.run_vanilla_ar(tgt, prompt, 64, want_jsonl=False)
    print(f"{dname}/{tname}: DOUBLE {len(r.output) / r.metrics['device_ms'] * 1e3:.1f} tok/s, AR "
          f"{len(a.output) / a.metrics['device_ms'] * 1e3:.1f} tok/s, lossless {r.output == a.output}", flush=True)
    del tgt, drf, st, r, a
    gc.collect()
