"""The NCCL slab path on real GPUs (tools/multigpu_check.py under torchrun): runs when at least
two CUDA devices are visible, skips otherwise (the round-end GPU tier has one)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("nproc", [2, 4, 8])
def test_nccl_slab_path_bitwise(nproc):
    n = _ngpu()
    if n < nproc:
        pytest.skip(f"needs {nproc} GPUs, {n} visible")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
                        "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc),
                        os.path.join(ROOT, "tools", "multigpu_check.py")], cwd=ROOT, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0 and "MULTIGPU_CHECK PASS" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
