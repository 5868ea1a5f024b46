"""Device timeline of the GEMMs of one target forward (DBL_GEMM_TRACE=1, DBL_GRAPHS=0):
per launch: first CTA resident, dependency resolved, last load issued, last epilogue done."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2601_05524_b200 as dbl  # noqa: E402
from paper_2601_05524_b200 import _capi  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-14b"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m = dbl.Transformer(dbl.transformer_config(name, seed=1, max_seq=1024))
L = _capi.lib()
out = (C.c_double * 8)()
_capi.check(L.dbl_profile_forward(m._h, 300, rows, 1, out))  # warm-up + passes (traced)
cap = 4096 * 320 * 4
st = np.zeros(cap, np.uint64)
grids = np.zeros(4096, np.int32)
byt = np.zeros(4096, np.int64)
n = C.c_int()
_capi.check(L.dbl_debug_gemm_trace(st.ctypes.data_as(C.POINTER(C.c_uint64)), cap,
                                   grids.ctypes.data_as(C.POINTER(C.c_int32)),
                                   byt.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
N = n.value
per = 161 if name == "qwen3-14b" else (28 * 4 + 1)
first = N - 2 * per  # pass 1 of profile_forward (no per-GEMM events)
st = st[:N * 320 * 4].reshape(N, 320, 4).astype(np.int64)
t0 = None
prev_end = None
tot_gap = tot_stream = 0
lines = []
for i in range(first, first + per):
    g = grids[i]
    s = st[i, :g]
    start, dep0, dep1 = s[:, 0].min(), s[:, 1].min(), s[:, 1].max()
    issued, end = s[:, 2].max(), s[:, 3].max()
    if t0 is None:
        t0 = start
    gap = (start - prev_end) if prev_end is not None else 0
    dur = end - dep1
    lines.append((i - first, g, byt[i] / 1e6, (start - t0) / 1e3, (dep1 - start) / 1e3, (issued - dep1) / 1e3,
                  (end - issued) / 1e3, dur / 1e3, byt[i] / max(dur, 1), gap / 1e3))
    prev_end = end
print(f"{'#':>3} {'grid':>4} {'MB':>7} {'t0 us':>8} {'wait':>6} {'stream':>7} {'drain':>6} {'dur':>6} {'GB/s':>6} {'gap':>6}")
for ln in lines[:12] + lines[-6:]:
    print("%3d %4d %7.1f %8.1f %6.1f %7.1f %6.1f %6.1f %6.0f %6.1f" % ln)
arr = np.array([ln[4:] for ln in lines])
print("mean wait %.2f stream %.2f drain %.2f dur %.2f us; sum dur %.1f us; total span %.1f us" % (
    arr[:, 0].mean(), arr[:, 1].mean(), arr[:, 2].mean(), arr[:, 3].mean(), arr[:, 3].sum(),
    (prev_end - t0) / 1e3))
