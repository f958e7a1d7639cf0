"""GPU: the multi-rank path of bench.py end to end on one device. Two ranks
(torchrun, gloo barriers, --same-device) each render their 64x64 super-tiles of
the C4 frame; rank 1 maps rank 0's framebuffer through CUDA IPC and stores its
pixels there; rank 0 checks the composed frame against its own single-device
render of the same animation time (multi_gpu_frame_identical). On a multi-GPU
box the same code runs with one device per rank and NVLink peer stores."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("compose,port,flag", [("ipc", 29531, True), ("gather", 29532, True), ("ipc", 29533, False)])
def test_two_ranks_compose_the_single_device_frame(gpu, compose, port, flag):
    """ipc: peer stores into rank 0's framebuffer; gather: the fallback without
    CUDA IPC (tiles packed per rank, collective gather, unpacked on rank 0).
    Without --same-device the bench finds the ranks share one GPU (GPU ids
    exchanged before the backend is chosen) and takes the same path."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-extras"] + (["--same-device"] if flag else [])
    env = dict(os.environ)
    if compose == "gather":
        env["VOXANIM_COMPOSE"] = "gather"
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["run"]["composition"].startswith("CUDA IPC stores" if compose == "ipc" else "collective gather")
    assert "sharing one GPU" in d["run"]["partition"]
    assert d["multi_gpu_frame_identical"] is True
    assert d["e2e"] is not None and d["e2e"]["value"] > 0
    # ranks sharing one GPU run the flag protocol with host polls (never device waits)
    assert d["run"]["frame_sync"].startswith("host-polled flags" if compose == "ipc" else "host synchronisation")
    assert d["frame_sync_timed_out"] in (None, False)


def test_bench_launches_its_own_ranks(gpu):
    """`bench.py --gpus 2` without a launcher starts two ranks itself (torch.distributed.run
    on 127.0.0.1) and reports n_gpus 2 and the composed frame's identity."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--same-device", "--steps", "3",
           "--warmup", "3", "--no-cpu-baseline", "--no-extras", "--e2e-steps", "5"]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=dict(os.environ))
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["multi_gpu_frame_identical"] is True
