"""Multi-GPU parity through torchrun + NCCL, when the box has
>= 2 GPUs: every rank's leaves after partitioned steps equal the single-process
golden states (uniform Sedov / smooth, AMR with cross-rank reflux), dt equal.
Skipped on single-GPU boxes (the gloo world-size-2/3 tests cover the host
logic on CPU)."""

import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("halo,xfer", [("p2p", "mapped"), ("p2p", "mapped-tail"), ("nccl", "threads-tail")])
@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_steps_match_single_process(world, halo, xfer):
    """halo: uniform trees read neighbour leaves over NVLink peer memory (default) or exchange
    them with NCCL (OMB_HALO=nccl); AMR trees always exchange.  xfer: the host transfers --
    the GPU reading / writing the mapped pinned leaves (after the step, or each launch part of
    the last stage written back while the next computes: -tail, small parts), or host threads
    around DMA copies with the download overlapped the same way."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(world), "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(HERE, "gpu_dist_check.py")]
    env = dict(os.environ, OMB_HALO=halo, OMB_HOST_XFER=xfer.split("-")[0])
    if xfer.endswith("-tail"):
        env["OMB_TAIL_RUNS"] = "2"
    else:
        env["OMB_TAIL_WAVES"] = "0"
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert f"multi-GPU parity on {world} ranks: OK" in r.stdout + r.stderr
