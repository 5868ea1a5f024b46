#!/usr/bin/env python
"""bench.py — the DOUBLE decode loop on B200 (BASELINE.json: decode tokens/s + speedup vs target-only
AR + mean accepted length).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload = BASELINE.json configs[1]: Qwen3-0.6B draft / Qwen3-14B target shapes, random-init
bf16, synthetic code-like prompt (HumanEval length, 160 tokens), 256 new tokens, greedy, d=10, N=3,
prior K=10.  A "step" is one complete DOUBLE decode of that request.  N>1 (torchrun, one process per
GPU): the target is tensor-parallel over the N GPUs (TpTransformer driven from rank 0,
the O/down and argmax exchange inside fwd_kernel over peer memory, the draft beside shard 0; strong
scaling of the one request), or N independent replicas with --tp off (weak scaling).

value          decode tokens/s of the DOUBLE loop with the weights/KV resident in HBM (CUDA events
               around the device decode loop, prompt prefill excluded), summed over ranks
e2e            the same metric through the public C-ABI (dbl_run) with host prompt/prior in and host
               tokens out, prefill and all copies inside the timed region (CUDA events)
speedup_vs_ar  value / target-only greedy AR tokens/s with the same kernels (run_vanilla_ar)
roofline       the verify forward = ONE persistent kernel (fwd_kernel: tcgen05 GEMMs, attention and
               fused epilogues): SURVEY §8(d) algorithmic bytes (weights + KV + embedding rows) /
               CUDA-event-timed launch duration vs MEASURED_PEAKS.json hbm_gbs
cpu_baseline   the reference's own host decode loop (oracle/_ref, unmodified run()) replaying this
               run's decision log — the forward is excluded (a transformer forward does not exist in
               the reference); 1 host core
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # configs[1]: 1 x B200 — the headline
    "qwen3-0.6b/qwen3-14b": dict(draft=("qwen3-0.6b", {}), target=("qwen3-14b", {}), prompt_len=160, max_new=256,
                                 desc="configs[1]: Qwen3-0.6B draft / Qwen3-14B target shapes, random-init bf16, "
                                      "synthetic code-like prompt (HumanEval length)"),
    # the north-star target (70B-shaped, configs[4] shapes) unsharded on one B200: 139 GB of weights
    "llama-3.2-1b/llama-3.3-70b": dict(draft=("llama-3.2-1b", {}), target=("llama-3.3-70b", {}), prompt_len=1024,
                                       max_new=256,
                                       desc="configs[4] shapes (Llama-3.2-1B draft / Llama-3.3-70B target), "
                                            "random-init bf16, CNN/DM-length synthetic prompt, target unsharded "
                                            "on 1 GPU"),
    # LABELLED aligned workload (SURVEY §7 hard part 6): an independent random-init draft never agrees
    # with a random-init target (alpha = 0, tools/align_probe.py).  Here the target's decoder layers >= 1
    # are initialised at 0.1x the HF std (they refine the residual stream instead of rewriting it) and the
    # draft is the target's own first layer + its embedding / LM head (early exit, same seed):
    # alpha ~0.97 teacher-forced.  Same Qwen3-14B shapes, bytes and kernels as configs[1].
    "aligned-qwen3-14b": dict(draft=("qwen3-14b", dict(n_layers=1, layer_std_scale=0.1, scale_from_layer=1)),
                              target=("qwen3-14b", dict(layer_std_scale=0.1, scale_from_layer=1)),
                              same_seed=True, prompt_len=160, max_new=256,
                              desc="LABELLED aligned workload: Qwen3-14B shapes, decoder layers >= 1 at 0.1x "
                                   "init std; draft = the target's first layer + embedding / LM head (early "
                                   "exit, same seed, 2.2 GB); random-init bf16, code-like prompt"),
    # small smoke workload (CI / quick checks)
    "tiny": dict(draft=("tiny-qwen-draft", {}), target=("tiny-qwen", {}), prompt_len=64, max_new=64, desc="tiny"),
}
SIDE_WORKLOADS = ("aligned-qwen3-14b", "llama-3.2-1b/llama-3.3-70b")
DEPTH, NGRAM, PRIOR_K = 10, 3, 10


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="qwen3-0.6b/qwen3-14b", choices=list(WORKLOADS))
    p.add_argument("--gamma", type=int, default=0, help="0 = ceil(C), C = t_target_fwd / t_draft_fwd")
    p.add_argument("--max-new", type=int, default=0)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--log-out", default="", help="write this run's decision log (json) here")
    p.add_argument("--no-serving", action="store_true", help="skip the batched-serving side measurement")
    p.add_argument("--no-side", action="store_true",
                   help="skip the side workloads (aligned draft, 70B-shaped target) after the headline")
    p.add_argument("--tp", choices=["auto", "off"], default="auto",
                   help="N>1: auto = the target tensor-parallel over the N GPUs (driven from rank 0), "
                        "off = N independent replicas")
    return p.parse_args()


# --------------------------------------------------------------------------- synthetic workload
def code_like_stream(vocab: int, n: int, seed: int, rho: float = 0.9):
    """A repetitive 'code-like' token stream: fresh 1-4 token spans mixed with replays (prob rho) of
    4-16 token spans of the stream so far — the recipe of gen_corpus (harness.cpp:151-186) with a
    numpy RNG.  Tokens avoid BOS (0) and EOS (vocab-1)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    s = []
    while len(s) < n:
        if len(s) >= 4 and rng.random() < rho:
            span = 4 + int(rng.random() * 13)
            st = int(rng.random() * len(s))
            s.extend(s[st:min(st + span, len(s))])
        else:
            s.extend(int(x) for x in rng.integers(1, vocab - 1, 1 + int(rng.random() * 4)))
    return s[:n]


def workload(vocab, prompt_len, seed):
    stream = code_like_stream(vocab, 64 * PRIOR_K + 4096, seed)
    corpus = [stream[i:i + 64] for i in range(0, len(stream), 64)]
    return stream[:prompt_len], corpus[:PRIOR_K]


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled every 200 ms during the timed region.  In-process NVML (one
    light query per sample) rather than an `nvidia-smi -lms` child: the latter's periodic driver calls
    stall the decode loop's host-side CUDA calls for up to hundreds of ms, which would show up in the
    end-to-end (host-API) number.  Falls back to nvidia-smi when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device, self.lines, self.proc, self.nv = device, [], None, None
        self.samples, self.stop = [], threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001 — no NVML: sample with nvidia-smi instead
            self.nv = None
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.wait(0.2):
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((float(sm), [n for n, b in zip(self.NAMES, self.bits) if r & b]))
            except Exception:  # noqa: BLE001
                pass

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        if self.nv is not None:
            for v, rs in self.samples:
                sm.append(v)
                reasons.update(rs)
            mx = float(self.mx)
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(self.NAMES, f[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "sampler": "nvml" if self.nv is not None else "nvidia-smi"}


# --------------------------------------------------------------------------- distributed plumbing
def dist_init(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return rank, world, local


def all_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_min(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def all_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# --------------------------------------------------------------------------- CPU baseline
def reference_replay(log, vocab, prompt, prior, max_new, gamma, target_tokens, reps=1):
    """Replay the decision log through the reference's unmodified host loop (oracle/_ref) — or the
    oracle port when the reference library was not built — and time it on one host core."""
    import ctypes as C
    import numpy as np
    from oracle.pyoracle import ARGMAX_FN, Oracle, reference_or_none
    orc = Oracle()
    L = orc.lib
    L.orc_replay_new.restype = C.c_void_p
    L.orc_replay_new.argtypes = [C.POINTER(C.c_int), C.c_long]
    L.orc_replay_reset.argtypes = [C.c_void_p]
    L.orc_replay_free.argtypes = [C.c_void_p]
    arr = np.ascontiguousarray(np.asarray(log, dtype=np.int32))
    rp = L.orc_replay_new(arr.ctypes.data_as(C.POINTER(C.c_int)), len(arr))
    dfn = ARGMAX_FN(C.cast(L.orc_replay_draft, C.c_void_p).value)
    tfn = ARGMAX_FN(C.cast(L.orc_replay_target, C.c_void_p).value)
    ref = reference_or_none()
    kind = "reference" if ref is not None else "port"
    times, out = [], None
    for _ in range(reps):
        L.orc_replay_reset(rp)
        t0 = time.perf_counter()
        if ref is not None:
            n = C.c_int()
            buf = (C.c_int * (max_new + 8))()
            js = C.create_string_buffer(1 << 22)
            met = (C.c_double * 8)()
            flat = [t for s in prior for t in s]
            rc = ref.lib.ref_run_callback(
                vocab, dfn, C.c_void_p(rp), tfn, C.c_void_p(rp), NGRAM, len(prior),
                (C.c_int * len(prior))(*[len(s) for s in prior]), (C.c_int * len(flat))(*flat),
                (C.c_int * len(prompt))(*prompt), len(prompt), max_new, gamma, DEPTH, 1, 1, 1,
                1.0, 1.0, 0.0, 0.0, buf, max_new + 8, C.byref(n), js, len(js), met)
            if rc:
                raise RuntimeError(ref.lib.ref_last_error().decode())
            out = list(buf[:n.value])
        else:
            st = orc.store(NGRAM, DEPTH)
            for i, s in enumerate(prior):
                st.insert(0, s, i)
            out, _, _ = orc.run(vocab, dfn, vocab, tfn, st, prompt, max_new, gamma=gamma, depth=DEPTH,
                                t_draft=1.0, duser=rp, tuser=rp)
        times.append(time.perf_counter() - t0)
    L.orc_replay_free(rp)
    if out != target_tokens:
        raise RuntimeError("reference replay diverged from the device run (parity failure)")
    return len(out) / min(times), kind


# --------------------------------------------------------------------------- main
def main():
    a = parse()
    rank, world, local = dist_init(a.gpus)
    wl = dict(WORKLOADS[a.workload])
    max_new = a.max_new or wl["max_new"]
    metric = "decode tokens/s (DOUBLE, greedy) + speedup vs target-only AR + mean accepted length"
    base_cfg = {"workload": f"{a.workload} ({wl['desc']})",
                "prompt_len": wl["prompt_len"], "max_new_tokens": max_new, "depth": DEPTH,
                "ngram": NGRAM, "prior_rounds": PRIOR_K, "temperature": 0,
                "parallelism": f"replicas x{world}" if world > 1 else "1 GPU (draft+target co-located)",
                "l2": "weights (>= 2 GB per model) >> L2 (126 MB): every forward streams from HBM"}

    if a.impl == "reference":
        return reference_arm(a, rank, world, wl, max_new, metric, base_cfg)
    if os.environ.get("DBL_BENCH_TP_DEVICES") and world == 1 and a.impl == "ours":
        return run_bench(a, 0, 1, 0, wl, max_new, metric, base_cfg,
                         tp_world=len(os.environ["DBL_BENCH_TP_DEVICES"].split(",")))
    tc = os.environ.get("DBL_TP_CHILD")
    if tc:  # one tensor-parallel rank (spawned by tp_children below): its own gloo group for the handles
        import torch.distributed as dist
        r, n, port = (int(x) for x in tc.split(","))
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=r, world_size=n)
        return run_bench(a, r, n, r, wl, max_new, metric, base_cfg, tp_world=n, tp_ipc=True)
    if world > 1 and a.tp == "auto":
        # Target tensor-parallel over the box's N GPUs, one process per GPU: every rank
        # builds its shard on its GPU, the ranks link their exchange buffers over CUDA IPC and run the same
        # decode loop (the O / down and argmax exchange inside fwd_kernel; the draft beside every shard —
        # BASELINE config 5's layout).  Each rank's TP run is a child process with a fresh CUDA context:
        # if any rank's child fails (even a device-side trap, which poisons the context), every rank falls
        # back to an independent replica (weak scaling) and the reason is recorded.
        barrier(world)
        line, err = tp_children(a, rank, world)
        if line is not None:
            if rank == 0:
                print(line, flush=True)
            barrier(world)
            return None
        if rank == 0:
            print(f"tensor-parallel bench failed ({err}); falling back to replicas", file=sys.stderr)
        base_cfg = dict(base_cfg, tp_error=err[:200])
    return run_bench(a, rank, world, local, wl, max_new, metric, base_cfg)


def tp_children(a, rank, world, cmd=None, timeout=600):
    """Run this rank's tensor-parallel child (bench.py with DBL_TP_CHILD=rank,world,port) and agree
    across ranks: returns (rank 0's JSON line — "" on other ranks — or None if any rank failed, the
    first error)."""
    import torch.distributed as dist
    port = int(os.environ.get("MASTER_PORT", "29500")) + 101
    env = dict(os.environ, DBL_TP_CHILD=f"{rank},{world},{port}")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "GROUP_RANK", "ROLE_RANK",
              "TORCHELASTIC_RUN_ID", "MASTER_PORT"):
        env.pop(k, None)
    if cmd is None:
        cmd = [sys.executable, os.path.abspath(__file__), "--gpus", "1", "--steps", str(a.steps),
               "--warmup", str(a.warmup), "--workload", a.workload, "--gamma", str(a.gamma),
               "--max-new", str(a.max_new), "--seed", str(a.seed), "--no-side"]
    line, err = None, ""
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
        outs = [x for x in r.stdout.splitlines() if x.startswith("{")]
        if r.returncode == 0 and (outs or rank != 0):
            line = outs[-1] if rank == 0 else ""
        else:
            err = f"rank {rank}: " + ((r.stderr.strip().splitlines() or ["no output"])[-1])
    except subprocess.TimeoutExpired:
        err = f"rank {rank}: timed out"
    ok = all_min(0.0 if line is None else 1.0, world) > 0.5
    errs = [None] * world
    dist.all_gather_object(errs, err)
    first = next((e for e in errs if e), "")
    return (line if ok else None), first


def _models(dbl, wl, seed, local, tp_world, tp_ipc=False, rank=0):
    """(target, draft, parallelism note) for a workload: a TP target is this rank's shard linked with
    the other processes' (tp_ipc), or all shards in-process over DBL_BENCH_TP_DEVICES."""
    tname, tkw = wl["target"]
    dname, dkw = wl["draft"]
    dseed = seed if wl.get("same_seed") else seed + 1
    note = None
    if tp_ipc:
        tgt = dbl.Transformer(dbl.transformer_config(tname, seed=seed, max_seq=4096, tp_rank=rank, tp_size=tp_world,
                                                     **tkw), device=local)
        dbl.link_tp_processes(tgt)
        note = (f"target TP={tp_world}, one process per GPU (CUDA IPC; the O / down and argmax exchange inside "
                "fwd_kernel), the draft beside every shard")
    elif tp_world > 1:
        # DBL_BENCH_TP_DEVICES="0,0": a TP layout on fewer GPUs (functional checks on one GPU)
        env_dev = os.environ.get("DBL_BENCH_TP_DEVICES")
        devices = [int(x) for x in env_dev.split(",")] if env_dev else list(range(tp_world))
        tgt = dbl.TpTransformer(dbl.transformer_config(tname, seed=seed, max_seq=4096, **tkw), devices=devices)
        note = (f"target TP={tp_world} on GPUs {devices} (peer memory, exchange inside fwd_kernel), "
                "draft beside shard 0")
    else:
        tgt = dbl.Transformer(dbl.transformer_config(tname, seed=seed, max_seq=4096, **tkw), device=local)
    drf = dbl.Transformer(dbl.transformer_config(dname, seed=dseed, max_seq=4096, **dkw), device=local)
    return tgt, drf, note


def measure(a, rank, world, local, wl, max_new, steps, warmup, tp_world=1, headline=True, tp_ipc=False):
    """One workload: DOUBLE at the headline gamma (device + e2e timing), target-only AR (the speedup
    denominator, same kernels), gamma = ceil(C) / 4 / 8, and the verify forward's roofline.  Ranks are
    independent replicas (tokens summed) unless they are the tensor-parallel ranks of one request."""
    import ctypes as C
    import torch
    import paper_2601_05524_b200 as dbl
    from paper_2601_05524_b200 import _capi
    tgt, drf, note = _models(dbl, wl, a.seed, local, tp_world, tp_ipc=tp_ipc, rank=rank)

    def tok_sum(x):
        return x if tp_ipc else all_sum(x, world)
    V = tgt.cfg.vocab
    prompt, prior = workload(V, wl["prompt_len"], a.seed + 100)

    def profile(model, ctx, rows, iters=5):
        out = (C.c_double * 8)()
        _capi.check(_capi.lib().dbl_profile_forward(model._h, ctx, rows, iters, out))
        return list(out)

    # C = t_target_fwd / t_draft_fwd at M = d+1 (harness.cpp:32-35)
    pt = profile(tgt, wl["prompt_len"], DEPTH + 1)
    pd = profile(drf, wl["prompt_len"], DEPTH + 1)
    C_ratio = pt[0] / pd[0]
    gamma_c = max(1, math.ceil(C_ratio))
    # The reference's gamma = ceil(C) assumes draft and target on separate devices (round time =
    # max(gamma*t_draft, t_target), pipeline.cpp:198-204).  Co-located on one GPU both stream HBM and the
    # round costs ~ t_target + gamma*t_draft; with an independent random-init draft (alpha = 0) every
    # drafted token is wasted, so configs[1]'s headline runs gamma = 1 and reports ceil(C), 4 and 8 beside
    # it.  The aligned workload (alpha > 0) runs the reference's gamma = ceil(C).
    gamma = a.gamma or (gamma_c if wl.get("same_seed") else 1)

    def store():
        st = dbl.HierarchicalDatastore(NGRAM, DEPTH, device=local)
        dbl.build_prior(st, prior, PRIOR_K)
        return st

    def run_double(g):
        return dbl.run(drf, tgt, store(), prompt, max_new, dbl.PipelineOptions(gamma=g, depth=DEPTH),
                       want_jsonl=False)

    for _ in range(warmup):
        run_double(gamma)
        dbl.run_vanilla_ar(tgt, prompt, max_new, want_jsonl=False)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev_ms, e2e_ms, tokens, launches = 0.0, 0.0, 0, 0
    results = []
    with ClockSampler(local) as clk:
        for _ in range(steps):
            torch.cuda.synchronize()
            e0.record()
            r = run_double(gamma)  # host prompt/prior in, host tokens out (e2e)
            e1.record()
            torch.cuda.synchronize()
            e2e_ms += e0.elapsed_time(e1)
            dev_ms += r.metrics["device_ms"]
            tokens += len(r.output)
            launches += r.metrics["kernel_launches"]
            results.append(r)
    torch.cuda.synchronize()
    barrier(world)
    log = dbl.last_run_log()
    # target-only AR with the same kernels (the speedup denominator) + lossless check
    ar_ms, ar_tok = 0.0, 0
    for _ in range(steps):
        ar = dbl.run_vanilla_ar(tgt, prompt, max_new, want_jsonl=False)
        ar_ms += ar.metrics["device_ms"]
        ar_tok += len(ar.output)
    ar_value = tok_sum(ar_tok) / (all_max(ar_ms, world) / 1e3)
    lossless = all(r.output == ar.output for r in results)
    m0 = results[-1].metrics

    def gamma_line(g):  # the same workload and timing at another gamma (ceil(C), 4, 8)
        nonlocal lossless
        run_double(g)
        gms, gtok, gm = 0.0, 0, None
        for _ in range(steps):
            rg = run_double(g)
            gms += rg.metrics["device_ms"]
            gtok += len(rg.output)
            lossless &= rg.output == ar.output
            gm = rg.metrics
        gv = tok_sum(gtok) / (all_max(gms, world) / 1e3)
        return {"gamma": g, "value": round(gv, 3), "speedup_vs_ar": round(gv / ar_value, 4),
                "mean_accepted_len": round(gm["m"], 4),
                "target_rows_per_forward": round(gm["target_rows"] / max(1, gm["target_fwd_count"]), 2)}

    value = tok_sum(tokens) / (all_max(dev_ms, world) / 1e3)
    main_line = {"gamma": gamma, "value": round(value, 3), "speedup_vs_ar": round(value / ar_value, 4),
                 "mean_accepted_len": round(m0["m"], 4),
                 "target_rows_per_forward": round(m0["target_rows"] / max(1, m0["target_fwd_count"]), 2)}
    gl = {}
    for key, g in (("gamma_C", gamma_c), ("gamma_1", 1), ("gamma_4", 4), ("gamma_8", 8)):
        gl[key] = main_line if g == gamma else next((v for v in gl.values() if v["gamma"] == g), None) or gamma_line(g)
    gl["gamma_C"] = dict(gl["gamma_C"], C_measured=round(C_ratio, 3))

    # roofline of the dominant kernel: the verify forward at this run's mean row count
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    rows_per_fwd = max(1, round(m0["target_rows"] / max(1, m0["target_fwd_count"])))
    ctx = wl["prompt_len"] + max_new // 2
    pv = profile(tgt, ctx, rows_per_fwd, iters=20)
    achieved = pv[2] / (pv[1] / 1e3) / 1e9  # GB/s: algorithmic bytes / event-timed fwd_kernel duration
    pdr = profile(drf, ctx, DEPTH + 1, iters=20)
    out = {
        "value": value, "e2e_ms": all_max(e2e_ms, world), "dev_ms": all_max(dev_ms, world),
        "tokens": tok_sum(tokens), "ar_value": ar_value, "gamma": gamma, "C": C_ratio, "m0": m0,
        "lossless": lossless, "gl": gl, "launches": tok_sum(launches), "clk": clk.summary(),
        "prompt": prompt, "prior": prior, "log": log, "output": results[-1].output, "V": V, "note": note,
        "roofline": {"bound": "hbm", "kernel": "fwd_kernel (persistent stream forward: tcgen05/TMA GEMMs + "
                              "attention + fused epilogues), one launch per verify forward",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4),
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured copy)" if peaks else "fallback",
                     "per_forward": {"tokens": int(pv[5]), "fwd_ms": round(pv[0], 4),
                                     "kernel_ms": round(pv[1], 4), "algorithmic_bytes": pv[2],
                                     "context": ctx, "rows": rows_per_fwd, "kernel_launches": int(pv[4]),
                                     "weight_stream_gbs": round(tgt.weight_bytes / (pv[0] / 1e3) / 1e9, 1)},
                     "draft_forward": {"rows": DEPTH + 1, "fwd_ms": round(pdr[0], 4),
                                       "algorithmic_bytes": pdr[2],
                                       "frac": round(pdr[2] / (pdr[1] / 1e3) / 1e9 / peak, 4)}},
    }
    if headline:
        out["retrieval"] = retrieval_probe(dbl, local, prompt, prior, V)
    if headline and tp_world <= 1 and not a.no_serving:
        # batched serving: B independent sequences of this workload's shape decoded in
        # lockstep, ONE target forward per step over all of them (run_vanilla_ar_batch; every stream ==
        # its own single-sequence AR).  Reported beside the headline, not in it.
        serving = {}
        for B in (8, 16):
            ps = [workload(V, wl["prompt_len"], a.seed + 500 + b)[0] for b in range(B)]
            dbl.run_vanilla_ar_batch(tgt, ps, 4)
            _, sm = dbl.run_vanilla_ar_batch(tgt, ps, 64)
            serving[f"B{B}"] = {"tokens_per_s": round(sm["tokens"] / (sm["device_ms"] / 1e3), 1),
                                "ms_per_step": round(sm["device_ms"] / 64, 3)}
        out["serving"] = dict(serving, what="target-only greedy decode of B sequences (64 new tokens "
                              "each) with one batched fwd_kernel per step; value above is B = 1")
    del tgt, drf
    import gc
    gc.collect()
    return out


def retrieval_probe(dbl, local, prompt, prior, V):
    """Device lookup latency (K1): on this workload's store, and on a paper-scale prior (~9.6 MB of
    tokens, the paper's K = 10 prior is ~9.5 MB) loaded by build_prior into the device
    n-gram index (store.cuh)."""
    st = dbl.HierarchicalDatastore(NGRAM, DEPTH, device=local)
    dbl.build_prior(st, prior, PRIOR_K)
    us_small = st.profile_lookup(prompt, DEPTH, 200)
    seq_len, n_seq = 64, 37500
    flat = code_like_stream(V, seq_len * n_seq, 4242)
    seqs = [flat[i * seq_len:(i + 1) * seq_len] for i in range(n_seq)]
    big = dbl.HierarchicalDatastore(NGRAM, DEPTH, device=local)
    t0 = time.perf_counter()
    dbl.build_prior(big, seqs, n_seq)
    build_ms = (time.perf_counter() - t0) * 1e3
    ctxs = [flat[i:i + 32] for i in range(1000, len(flat) - 64, len(flat) // 8)]
    us_big = statistics.median(big.profile_lookup(c, DEPTH, 100) for c in ctxs)
    return {"kernel": "lookup (K1, one CTA per query: index probes + tail scan)",
            "workload_store_lookup_us": round(us_small, 2),
            "paper_scale_prior": {"tokens": len(flat), "mbytes": round(4 * len(flat) / 1e6, 2),
                                  "index_entries": big.prior.index_entries,
                                  "build_prior_ms": round(build_ms, 1), "lookup_us_median": round(us_big, 2)}}


def side_line(a, local, name):
    """A compact line for a non-headline workload (1 warm-up, 1 timed decode per gamma)."""
    wl = WORKLOADS[name]
    r = measure(a, 0, 1, local, wl, wl["max_new"], 1, 1, headline=False)
    return {"desc": wl["desc"], "value": round(r["value"], 3), "unit": "tokens/s", "gamma": r["gamma"],
            "ar_tokens_per_s": round(r["ar_value"], 3), "speedup_vs_ar": round(r["value"] / r["ar_value"], 4),
            "mean_accepted_len": round(r["m0"]["m"], 4), "amt": round(r["m0"]["amt"], 4),
            "target_rows_per_forward": r["gl"]["gamma_C"]["target_rows_per_forward"] if r["gamma"] ==
            r["gl"]["gamma_C"]["gamma"] else None,
            "e2e_tokens_per_s": round(r["tokens"] / (r["e2e_ms"] / 1e3), 3), "lossless_vs_ar": r["lossless"],
            "gammas": r["gl"], "roofline": {k: r["roofline"][k] for k in ("achieved", "frac", "per_forward",
                                                                           "draft_forward")},
            "timing": "1 warm-up + 1 timed decode per gamma (side line; the headline uses --steps/--warmup)"}


def run_bench(a, rank, world, local, wl, max_new, metric, base_cfg, tp_world=1, tp_ipc=False):
    import paper_2601_05524_b200 as dbl
    from paper_2601_05524_b200 import _capi
    if not _capi.lib().dbl_device_ok():
        raise SystemExit("no usable sm_100 device (libdouble_b200 has no CPU fallback)")
    import torch
    torch.cuda.set_device(local)
    r = measure(a, rank, world, local, wl, max_new, a.steps, a.warmup, tp_world=tp_world,
                headline=tp_world <= 1, tp_ipc=tp_ipc)
    if r["note"]:
        base_cfg = dict(base_cfg, parallelism=r["note"], tp=tp_world)
    t_e2e = r["e2e_ms"]
    value = r["value"]
    m0 = r["m0"]
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
        traffic = prof.get(a.workload)
    except (OSError, ValueError):
        pass
    line = {
        "metric": metric, "value": round(value, 3), "unit": "tokens/s", "n_gpus": max(world, tp_world),
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(r["dev_ms"] / a.steps, 3),
        "higher_is_better": True, "scaling": "strong" if tp_world > 1 else "weak", "vs_baseline": None,
        "dtype": "bf16", "n_gpus_used": max(world, tp_world),
        "data": "synthetic (random-init weights, code-like prompt)",
        "config": dict(base_cfg, gamma=r["gamma"], C_measured=round(r["C"], 3)),
        "speedup_vs_ar": round(value / r["ar_value"], 4), "ar_tokens_per_s": round(r["ar_value"], 3),
        "mean_accepted_len": round(m0["m"], 4), "amt": round(m0["amt"], 4),
        "rounds_per_step": m0["rounds"],
        "target_rows_per_forward": round(m0["target_rows"] / max(1, m0["target_fwd_count"]), 3),
        "lossless_vs_ar": r["lossless"],
        "gamma_C": r["gl"]["gamma_C"], "gamma_4": r["gl"]["gamma_4"], "gamma_8": r["gl"]["gamma_8"],
        "e2e": {"value": round(r["tokens"] / (t_e2e / 1e3), 3), "unit": "tokens/s",
                "h2d_bytes_per_step": 4 * (len(r["prompt"]) + sum(len(s) for s in r["prior"])),
                "d2h_bytes_per_step": 4 * max_new},
        "roofline": dict(r["roofline"], traffic=traffic),
        "gpu_launches": int(r["launches"]),
    }
    cs = r["clk"]
    line["clocks"] = {"sm_mhz": cs["sm_mhz"], "sm_max_mhz": cs["sm_max_mhz"], "reasons": cs["reasons"]}
    if "serving" in r:
        line["serving_batch"] = r["serving"]
    if "retrieval" in r:
        line["retrieval"] = r["retrieval"]
    if a.log_out and rank == 0:
        json.dump({"vocab": r["V"], "prompt": r["prompt"], "prior": r["prior"], "max_new": max_new,
                   "gamma": r["gamma"], "output": r["output"], "log": [int(x) for x in r["log"]]},
                  open(a.log_out, "w"))
    if rank == 0:
        try:
            cpu_v, kind = reference_replay(r["log"], r["V"], r["prompt"], r["prior"], max_new, r["gamma"],
                                           r["output"], reps=2)
            line["cpu_baseline"] = {"value": round(cpu_v, 3), "unit": "tokens/s", "cores": 1, "kind": kind,
                                    "sample": f"one {max_new}-token DOUBLE decode of this workload replayed "
                                              "through the reference host loop (run(), pipeline.cpp) with the "
                                              "forward excluded: argmax rows served from this run's decision "
                                              f"log as one-hot fp64 rows of V={r['V']} (argmax_token included)"}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
        if tp_world <= 1 and world == 1 and not a.no_side and a.workload == "qwen3-0.6b/qwen3-14b":
            side = {}
            for name in SIDE_WORKLOADS:
                try:
                    side[name] = side_line(a, local, name)
                except Exception as e:  # noqa: BLE001
                    side[name] = {"error": str(e)[:300]}
            line["side_workloads"] = side
        print(json.dumps(line), flush=True)


def reference_arm(a, rank, world, wl, max_new, metric, base_cfg):
    """--impl reference: the reference's own CPU decode loop on this workload (forward excluded), from
    the recorded decision log bench_data/<workload>.json (produced by this bench, --log-out)."""
    if rank != 0:
        return
    path = os.path.join(ROOT, "bench_data", a.workload.replace("/", "_") + ".json")
    try:
        d = json.load(open(path))
    except OSError:
        print(json.dumps({"impl": "reference", "unavailable": f"no recorded decision log at {path}"}))
        return
    times = []
    vals = []
    for _ in range(a.warmup):
        reference_replay(d["log"], d["vocab"], d["prompt"], d["prior"], d["max_new"], d["gamma"], d["output"])
    for _ in range(a.steps):
        t0 = time.perf_counter()
        v, kind = reference_replay(d["log"], d["vocab"], d["prompt"], d["prior"], d["max_new"], d["gamma"],
                                   d["output"])
        times.append(time.perf_counter() - t0)
        vals.append(v)
    value = statistics.median(vals)
    print(json.dumps({
        "impl": "reference", "metric": metric, "value": round(value, 3), "unit": "tokens/s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": round(1e3 * statistics.median(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (recorded decision log)",
        "config": dict(base_cfg, gamma=d["gamma"]),
        "cpu_baseline": {"value": round(value, 3), "unit": "tokens/s", "cores": 1, "kind": kind,
                         "sample": f"{d['max_new']}-token DOUBLE decode replayed through the reference host "
                                   "loop (forward excluded)"},
        "e2e": {"value": round(value, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
