"""One process per GPU (torchrun + NCCL): per-rank tables bit-exact against
the golden fixtures and the merged raster identical to the reference's.
Needs >= 2 GPUs (run with `gpurun --gpus 2` / `--gpus 4`)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu

CASES = {
    2: ["balanced_2r_p2p", "balanced_2r_sparse_coll", "explicit_2r_coll", "multi_area_2r", "multi_area_2r_coll",
        "poisson_multi_p2p", "poisson_multi_coll", "no_multapse_p2p", "no_multapse_coll"],
    3: ["remote_p2p", "remote_coll", "explicit_3r_p2p", "explicit_3r_coll", "dist_random_p2p", "dist_random_coll"],
    4: ["balanced_4r_p2p", "balanced_4r_coll"],
}


@pytest.mark.parametrize("world", sorted(CASES))
def test_multiprocess(world):
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29531", os.path.join(HERE, "mp_worker.py"), *CASES[world]]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
