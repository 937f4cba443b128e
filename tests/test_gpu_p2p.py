"""PCMM reduce-scatter over CUDA IPC / NVLink peer memory in real separate
processes on one GPU (same-device IPC): the executor's own data plane (device
mode: comm stream, pushes + flags in the windows, no host in the loop;
dist.attach_p2p) and the host-synchronised hook (dist.P2pReducer).
N = 2^11, T = 64 has 4 token groups (the T = 2048, N = 2^16 structure), so
world 8 / 16 puts 2 / 4 ranks on each group.  Bundle hashes summed over the
ranks must equal the unsharded run, with the peer-memory path actually used."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,tokens,mode,kind,modes,stagger", [
    (8, 64, "device", 0, 0, 0), (16, 64, "device", 0, 0, 0), (8, 64, "hook", 0, 0, 0), (2, 16, "device", 1, 0, 0),
    (8, 64, "device", 0, 1, 0), (2, 16, "device", 1, 1, 0), (8, 64, "device", 0, 0, 1), (8, 64, "device", 0, 1, 1)])
def test_p2p_reduce_scatter_processes(world, tokens, mode, kind, modes, stagger):
    """mode device: the executor's comm-stream exchange with flags in the IPC
    windows (no Python in the layer); hook: the host-synchronised reducer.
    kind 1: the FFN graph at T = 16 -- one token group split over 2 ranks.
    modes 1: matmuls gather or reduce as the reference's byte rule picks
    (all-gathers of the activation on the comm stream)."""
    env = dict(os.environ, P2P_TOKENS=str(tokens), P2P_MODE=mode, P2P_KIND=str(kind), P2P_MODES=str(modes),
               P2P_STAGGER=str(stagger))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "_p2p_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("P2P_")]
    assert line and line[0].startswith("P2P_OK") and "used_p2p=True" in line[0], r.stdout[-2000:] + r.stderr[-2000:]
    # the bytes the ranks actually sent are the plan's executed events (aegis_plan_*)
    kv = dict(t.split("=") for t in line[0].split()[1:])
    assert int(kv["sent"]) == int(kv["planned"]) > 0, line[0]


def test_p2p_dropped_exchange_is_detected():
    """Separate processes, device data plane, exchange dropped by fault
    injection: the summed hashes must differ from the unsharded run."""
    env = dict(os.environ, P2P_TOKENS="64", P2P_MODE="device", P2P_FAULT="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", "8",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "_p2p_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("P2P_")]
    assert line and line[0].startswith("P2P_MISMATCH"), r.stdout[-2000:]
    assert " sent=0 " in line[0], line[0]
