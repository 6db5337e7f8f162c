"""The slab driver with one PROCESS per rank (torchrun, gloo, every rank on GPU 0): the
bench's own DamBreakSlab / Exchanger / GpuBackend path with migration, halo values and
re-balancing equals a single-context run bitwise. The thread-rank test of
test_gpu_parity.py covers the rank logic; this one covers the process path — torch row
tensors, the exchange and the library's kernels ordered on one stream."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("world", [2, 3])
def test_slab_ranks_as_processes_match_plain(world, mode):
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "two_process_slab.py"), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "two_process_slab OK" in r.stdout


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("world", [2, 3])
def test_nbody_shards_as_processes_match_plain(world, mode):
    port = free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "two_process_slab.py"), mode, "nbody"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "two_process_slab OK" in r.stdout
