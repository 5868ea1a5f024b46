"""GPU (>= 2 GPUs): tensor parallel with ONE PROCESS PER SHARD (the contract's launch
model): two torchrun ranks, one GPU each, link their shards over CUDA IPC (handles all-gathered with
torch.distributed/gloo) and run the same decode loop; the exchange runs inside fwd_kernel.

Needs two GPUs: two processes' persistent forwards cannot share one GPU (a context holding tensor
memory is not time-sliced against another, so their exchange would wait forever).  The in-process
group (tests/test_gpu_tp.py) runs on the same model-level exchange buffers and tags; this test adds
the IPC handle exchange and the one-process-per-GPU launch."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_two_processes_one_shard_each():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one process per GPU needs >= 2 GPUs (this box has %d)" % torch.cuda.device_count())
    env = dict(os.environ, PYTHONPATH=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "tools", "tp_ipc_check.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("DOUBLE == AR True, identical on all ranks True") == 2, r.stdout[-2000:]
