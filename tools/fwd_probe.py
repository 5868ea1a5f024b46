"""Times one model's verify forward (profile_forward): python tools/fwd_probe.py MODEL ROWS CTX ITERS.
Environment knobs (DBL_FWD_SMEM_KB, DBL_FWD_DBG, ...) are read by the library at first use."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402
from paper_2601_05524_b200 import _capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-14b"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 300
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
m = dbl.Transformer(dbl.transformer_config(name, seed=1, max_seq=4096))
out = np.zeros(8)
_capi.check(_capi.lib().dbl_profile_forward(m._h, ctx, rows, iters, out.ctypes.data_as(_capi.F64P)))
print(f"{name} rows={rows} ctx={ctx} smem_kb={os.environ.get('DBL_FWD_SMEM_KB', 'default')} "
      f"fwd_ms={out[0]:.4f} GB/s={out[2] / out[0] / 1e6:.0f}")
