"""GPU: the frame-completion flags of the multi-GPU path (vxa_frame_open/close).

On N GPUs rank 0's stream opens a frame with a go flag and closes it with a
1-thread kernel that waits for every rank's done flag in its HBM; the other
ranks wait for go and store done after their frame (system-scope release /
acquire over NVLink). Kernels that wait on one another must never share a GPU,
so on this one-GPU box every device-side wait below is launched only after the
flag it waits for has been written (host-sequenced), and the timeout test waits
for a flag nobody writes. The concurrent protocol itself runs on one GPU with
host-polled flags (tests/test_gpu_multirank_bench.py).
"""
import ctypes as C
import multiprocessing as mp
import os
import sys
import time

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_wait_for_a_missing_rank_times_out_and_latches(gpu):
    import paper_1911_06001_b200 as vx
    from paper_1911_06001_b200 import _abi

    lib = vx.vxa()
    ctx = C.c_void_p()
    assert lib.vxa_create(0, C.byref(ctx)) == 0
    try:
        h = (C.c_char * 64)()
        assert lib.vxa_sync_export(ctx, 2, h) == 0
        assert lib.vxa_sync_configure(ctx, _abi.VXA_SYNC_DEVICE, 100) == 0
        to = C.c_int32()
        assert lib.vxa_sync_status(ctx, C.byref(to)) == 0 and to.value == 0
        t0 = time.perf_counter()
        assert lib.vxa_frame_open(ctx) == 0   # go = 1
        assert lib.vxa_frame_close(ctx) == 0  # waits for done[1] == 1: nobody writes it
        assert lib.vxa_synchronize(ctx) == 0
        assert time.perf_counter() - t0 < 5.0
        assert lib.vxa_sync_status(ctx, C.byref(to)) == 0 and to.value == 1
        # argument checks
        assert lib.vxa_sync_export(ctx, 1, h) == _abi.VXA_ERR_INVALID
        assert lib.vxa_sync_configure(ctx, 7, 0) == _abi.VXA_ERR_INVALID
    finally:
        lib.vxa_destroy(ctx)


def _rank(rank, q_in, q_out, frames):
    sys.path.insert(0, ROOT)
    os.environ["VOXANIM_DEVICE"] = "0"
    import paper_1911_06001_b200 as vx
    from paper_1911_06001_b200 import _abi

    lib = vx.vxa()
    ctx = C.c_void_p()
    assert lib.vxa_create(0, C.byref(ctx)) == 0
    h = (C.c_char * 64)()
    if rank == 0:
        assert lib.vxa_sync_export(ctx, 2, h) == 0
        q_out.put(bytes(h))
    else:
        got = q_in.get(timeout=60)
        assert lib.vxa_sync_import(ctx, 1, 2, (C.c_char * 64).from_buffer_copy(got)) == 0, lib.vxa_last_error()
    assert lib.vxa_sync_configure(ctx, _abi.VXA_SYNC_DEVICE, 5000) == 0
    for k in range(frames):
        if rank == 0:
            assert lib.vxa_frame_open(ctx) == 0          # go = k + 1
            assert lib.vxa_synchronize(ctx) == 0         # ... written before rank 1 waits on it
            q_out.put(("go", k))
            assert q_in.get(timeout=60) == ("done", k)   # rank 1's done flag is written
            assert lib.vxa_frame_close(ctx) == 0         # device wait, already satisfied
            assert lib.vxa_synchronize(ctx) == 0
        else:
            assert q_in.get(timeout=60) == ("go", k)
            assert lib.vxa_frame_open(ctx) == 0          # device wait, already satisfied
            assert lib.vxa_frame_close(ctx) == 0         # done[1] = k + 1
            assert lib.vxa_synchronize(ctx) == 0
            q_out.put(("done", k))
    to = C.c_int32()
    assert lib.vxa_sync_status(ctx, C.byref(to)) == 0 and to.value == 0
    lib.vxa_destroy(ctx)


def test_device_flags_between_two_processes(gpu):
    """Rank 1 maps rank 0's flag block through CUDA IPC; over 5 frames every
    device-side wait finds its flag (frame numbers agree on both sides) and no
    wait times out (each process asserts its own status and exits 0)."""
    mpc = mp.get_context("spawn")
    to0, to1 = mpc.Queue(), mpc.Queue()
    p0 = mpc.Process(target=_rank, args=(0, to0, to1, 5))  # reads to0, writes to1
    p1 = mpc.Process(target=_rank, args=(1, to1, to0, 5))
    p0.start()
    p1.start()
    p0.join(300)
    p1.join(300)
    for p in (p0, p1):
        if p.is_alive():
            p.kill()
    assert p0.exitcode == 0 and p1.exitcode == 0
