"""Multi-GPU parity: runs tests/dist_check.py under torchrun with one rank per
visible GPU (2 and, when present, 4). Needs >= 2 B200s; the CPU-side partition logic is
covered by tests/test_distribute.py (gloo, world_size 2)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("world,env", [(2, {}), (4, {}),
                                       # separate flag-based exchange kernels
                                       (2, {"BDDC_FUSED_EX": "0", "DIST_CHECK_C3": "0"}),
                                       (2, {"BDDC_P2P": "0", "DIST_CHECK_C3": "0"}),  # NCCL exchanges
                                       (2, {"BDDC_SPLIT": "0", "BDDC_HARMONIC": "0", "DIST_CHECK_C3": "0"})],
                         ids=["w2", "w4", "w2-exchange-kernels", "w2-nccl", "w2-unpruned"])
def test_distributed_matches_single_gpu_and_reference(gpu, world, env):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs (have {_gpus()})")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world + 10 * len(env)),
           os.path.join(ROOT, "tests", "dist_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=ROOT, env={**os.environ, **env})
    print(out.stdout[-4000:], out.stderr[-4000:])
    assert out.returncode == 0
