"""N>1 path on real GPUs: launches tools/dist_check.py under torchrun when at
least two GPUs are visible (gpurun --gpus 2/4); skipped on a single-GPU box.
Runs the default exchange, the producer-epilogue stores, NCCL, and the C-ABI
trainer (full graph and per-rank EAS subgraphs); the full 14-mode sweep is
tools/dist_check.py without --modes (profiles/r02_dist_check_n*.json).
The CPU side of the same exchange is covered by test_exchange_gloo.py."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_row_partitioned_training_matches_oracle():
    import torch
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    nproc = min(n, 4)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
                        "--master-port", "29531", os.path.join(ROOT, "tools", "dist_check.py"),
                        "--modes", "sm,epilogue,nccl,native,native-eas,native-fused,native-p24"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and line, r.stdout[-2000:] + r.stderr[-2000:]
    assert json.loads(line[-1])["ok"]
