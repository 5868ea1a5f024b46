"""Device timeline of one stream forward (DBL_FWD_TRACE=1): per phase, when its weights started
streaming, when its input dependency resolved and when its last contribution was signalled.

    DBL_FWD_TRACE=1 python tools/fwd_timeline.py [model] [rows] [ctx]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_05524_b200 as dbl  # noqa: E402
from paper_2601_05524_b200 import _capi  # noqa: E402
from paper_2601_05524_b200.models import PRESETS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qwen3-14b"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = int(sys.argv[3]) if len(sys.argv) > 3 else 300
if os.environ.get("DBL_FWD_TRACE") != "1":
    print("note: DBL_FWD_TRACE!=1, timeline unavailable")
m = dbl.Transformer(dbl.transformer_config(name, seed=1, max_seq=max(1024, ctx + rows + 64)))
L = _capi.lib()
out = (C.c_double * 8)()
_capi.check(L.dbl_profile_forward(m._h, ctx, rows, 1, out))
if os.environ.get("DBL_FWD_TRACE") != "1":
    print(f"# {name}: rows={rows} ctx={ctx}; fwd {out[0]*1e3:.1f} us (event-timed)")
    sys.exit(0)
nl, h, f, nh, nkv, hd, V, tied, _, _ = PRESETS[name]
cap = (6 * nl + 8) * 160 * 16
st = np.zeros(cap, np.uint64)
n_ph, grid = C.c_int(), C.c_int()
_capi.check(L.dbl_debug_fwd_trace(st.ctypes.data_as(C.POINTER(C.c_uint64)), cap, C.byref(n_ph), C.byref(grid)))
P, G = n_ph.value, grid.value
st = st[:P * G * 16].reshape(P, G, 16).astype(np.int64)
per_layer = (P - 3) // nl  # 5 (attention combined by its last item) or 6 (a separate combine phase)
kinds, mb = ["embed"], [0.0]
for _ in range(nl):
    if per_layer == 6:
        kinds += ["qkv", "attn", "combine", "o", "gate|up", "down"]
        mb += [(nh + 2 * nkv) * hd * h * 2 / 1e6, 0.0, 0.0, h * nh * hd * 2 / 1e6, 2 * f * h * 2 / 1e6, h * f * 2 / 1e6]
    else:
        kinds += ["qkv", "attn", "o", "gate|up", "down"]
        mb += [(nh + 2 * nkv) * hd * h * 2 / 1e6, 0.0, h * nh * hd * 2 / 1e6, 2 * f * h * 2 / 1e6, h * f * 2 / 1e6]
kinds += ["lm_head", "argmax"]
mb += [V * h * 2 / 1e6, 0.0]
assert len(kinds) == P, (len(kinds), P)
valid = st > 0
t0 = st[valid].min()
rel = lambda x: (x - t0) / 1e3  # noqa: E731


def col(p, k, fn):
    v = st[p, :, k][st[p, :, k] > 0]
    return fn(v) if len(v) else 0


print(f"# {name}: rows={rows} ctx={ctx} grid={G}; fwd {out[0]*1e3:.1f} us (event-timed)")
print(f"{'#':>4} {'phase':>8} {'MB':>7} {'w0 us':>8} {'dep us':>8} {'done us':>8} {'dur':>6} {'GB/s':>6}")
prev_done = 0.0
tot = {}
for p in range(P):
    w0 = rel(col(p, 0, np.min)) if col(p, 0, np.min) else float("nan")
    dep = rel(col(p, 1, np.max)) if col(p, 1, np.max) else float("nan")
    done = rel(col(p, 2, np.max))
    dur = done - prev_done
    gbs = mb[p] * 1e6 / (dur * 1e3) if dur > 0 and mb[p] else 0
    tot.setdefault(kinds[p], [0.0, 0.0])
    tot[kinds[p]][0] += dur
    tot[kinds[p]][1] += mb[p]
    if p < 12 or p >= P - 8:
        print(f"{p:4d} {kinds[p]:>8} {mb[p]:7.1f} {w0:8.1f} {dep:8.1f} {done:8.1f} {dur:6.1f} {gbs:6.0f}")
    prev_done = done
print("per phase kind: total us / MB / GB/s")
for k, (us, b) in tot.items():
    print(f"  {k:>8} {us:9.1f} us {b:9.1f} MB {b * 1e6 / max(us * 1e3, 1):7.0f} GB/s")
print(f"span {prev_done:.1f} us; weights {sum(mb):.0f} MB -> {sum(mb) * 1e6 / (prev_done * 1e3):.0f} GB/s")

# ---- detail of one middle layer: per phase, percentiles over CTAs relative to the previous phase's end
L0 = 1 + per_layer * (nl // 2)
print(f"\nlayer {nl // 2} detail (us after the previous phase's last signal; min/median/max over CTAs)")
names = {1: "dep", 4: "mma0", 5: "mma1", 6: "epi1", 2: "sig"}
prev = col(L0 - 1, 2, np.max)
for p in range(L0, L0 + per_layer):
    parts = []
    for k in (1, 4, 5, 6, 2):
        v = st[p, :, k][st[p, :, k] > 0]
        if len(v):
            q = (np.percentile(v, [0, 50, 100]) - prev) / 1e3
            parts.append(f"{names[k]} {q[0]:6.1f}/{q[1]:6.1f}/{q[2]:6.1f}")
    print(f"  {kinds[p]:>8}: " + "  ".join(parts))
    prev = col(p, 2, np.max)

# ---- stragglers of the middle layer's GEMM phases: which CTAs finish their epilogue last, and why
sms = G
units, active, offset, kbs = {}, {}, {}, {}
off = 0
shapes = {"qkv": ((nh + 2 * nkv) * hd, h), "o": (h, nh * hd), "gate|up": (2 * f, h), "down": (h, f), "lm_head": (V, h)}
for p in range(P):
    if kinds[p] in shapes:
        n_out, K = shapes[kinds[p]]
        U = ((n_out + 127) // 128) * (K // 64)
        A = max(1, min(sms, U // 4))
        units[p], active[p], offset[p], kbs[p] = U, A, off, K // 64
        off = (off + A) % sms
print("\nstragglers (epilogue end - last MMA, us): top CTAs per phase")
for p in range(L0, L0 + per_layer):
    if p not in units:
        continue
    U, A, o, KB = units[p], active[p], offset[p], kbs[p]
    lag = (st[p, :, 6] - st[p, :, 5]) / 1e3
    wake = (st[p, :, 7] - st[p, :, 5]) / 1e3
    order = np.argsort(-lag)[:4]
    desc = []
    for c in order:
        ci = (c - o) % sms
        b0, b1 = ci * U // A, (ci + 1) * U // A
        sub = [(st[p, c, k] - st[p, c, 5]) / 1e3 for k in (7, 8, 9, 12, 13, 14, 15, 10, 11, 6)]
        desc.append(f"c{c}(ci{ci} tiles {b0 // KB}-{(b1 - 1) // KB}) {lag[c]:.1f} [acc/fin/fix/q0/q1/q2/q3/epi/sig/end " +
                    "/".join(f"{x:.1f}" for x in sub) + "]")
    print(f"  {kinds[p]:>8} median {np.median(lag):.1f}:\n      " + "\n      ".join(desc))

ap = L0 + 1  # the middle layer's attention phase (its combine follows)
w_end = st[ap, :, 8:12].max(axis=1)
prev_done = col(L0, 2, np.max)
print(f"\nattention (layer {nl // 2}): per-CTA last item done after QKV end: median "
      f"{(np.median(w_end) - prev_done) / 1e3:.1f} max {(w_end.max() - prev_done) / 1e3:.1f} us; "
      f"CTA signal max {(col(ap, 2, np.max) - prev_done) / 1e3:.1f} us; epilogue start median "
      f"{(np.median(st[ap, :, 3]) - prev_done) / 1e3:.1f}")

# attention item internals (middle layer): per CTA with an item, us after the CTA's phase start (stamp 3)
rows = []
for c in range(G):
    if st[ap, c, 15] > 0 and st[ap, c, 3] > 0:
        b = st[ap, c, 3]
        rows.append([(st[ap, c, k] - b) / 1e3 for k in (12, 13, 14, 15, 2)] + [(b - prev_done) / 1e3])
if rows:
    r = np.array(rows)
    print("attention items: loads/scores/softmax/item-end/signal after phase start, and phase start after QKV end"
          " (median / max over %d CTAs):" % len(rows))
    print("  " + "  ".join(f"{n} {np.median(r[:, i]):.1f}/{r[:, i].max():.1f}" for i, n in
                           enumerate(["loads", "scores", "softmax", "end", "signal", "start"])))
