"""One process per shard (run under torchrun, world 2..8): each rank links its tensor-parallel shard with
the others over CUDA IPC and runs the same decode loop.  Checks (exit code != 0 on failure):
  * the shard's logits columns == the unsharded model's within the bf16/fp32 tolerance, argmax rows
    identical on every rank;
  * DOUBLE with a table draft == target-only AR with the same TP target, identical on every rank.
Devices: DBL_TP_IPC_DEVICES="0,1,..." (default: rank r on GPU r; "same" = every rank on GPU 0)."""
import os
import random
import sys

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05524_b200 as dbl  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    spec = os.environ.get("DBL_TP_IPC_DEVICES", "")
    dev = 0 if spec == "same" else (int(spec.split(",")[rank]) if spec else rank)
    name = os.environ.get("DBL_TP_IPC_MODEL", "tiny-qwen")
    shard = dbl.Transformer(dbl.transformer_config(name, seed=3, max_seq=1024, tp_rank=rank, tp_size=world), device=dev)
    dbl.link_tp_processes(shard)
    full = dbl.Transformer(dbl.transformer_config(name, seed=3, max_seq=1024), device=dev)
    V, Vl = shard.cfg.vocab, shard.cfg.vocab // world
    rng = random.Random(5)
    ok = True
    for L, c in ((1, 0), (9, 4), (70, 10)):
        ctx = [rng.randrange(V) for _ in range(L)]
        cands = [rng.randrange(V) for _ in range(c)]
        a = dbl.forward_logits(full, ctx, cands)
        b = dbl.forward_logits(shard, ctx, cands)[:, rank * Vl:(rank + 1) * Vl]
        err = np.abs(a[:, rank * Vl:(rank + 1) * Vl] - b).max() / np.abs(a).max()
        am = dbl.forward_batch(shard, ctx, cands)
        rows = [None] * world
        dist.all_gather_object(rows, am)
        ok &= err <= 2e-2 and all(r == am for r in rows)
        print(f"rank {rank}: L={L} c={c} rel err {err:.2e} argmax rows equal on all ranks {all(r == am for r in rows)}",
              flush=True)
    prng = np.random.default_rng(12)
    probs = prng.random((V, V)) ** 8
    probs /= probs.sum(axis=1, keepdims=True)
    drf = dbl.TableModel(1, V, np.arange(V, dtype=np.int32), probs, np.full(V, 1.0 / V), device=dev)
    base = [rng.randrange(1, V - 1) for _ in range(40)]
    prior = [(base * 3)[i:i + 64] for i in range(0, 30, 3)]
    st = dbl.HierarchicalDatastore(3, 10, device=dev)
    dbl.build_prior(st, prior, 10)
    r = dbl.run(drf, shard, st, prior[0][:24], 64, dbl.PipelineOptions(gamma=2, depth=10))
    ar = dbl.run_vanilla_ar(shard, prior[0][:24], 64)
    outs = [None] * world
    dist.all_gather_object(outs, r.output)
    ok &= r.output == ar.output and all(o == r.output for o in outs)
    print(f"rank {rank}: DOUBLE == AR {r.output == ar.output}, identical on all ranks {all(o == r.output for o in outs)}",
          flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
