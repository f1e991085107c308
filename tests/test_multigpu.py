"""Multi-GPU parity: the torchrun scripts tests/mgpu_check.py (ladder / ring / hole-hole
with split and round-robin ownership, bitwise equal to 1 GPU and within 1e-11 of the oracle; scalar
all-reduce; permuted add; implicit Cholesky ladder) and tests/mgpu_ccsd_check.py (the CCSD-shaped
iteration with distributed placement and compact R2 vs the oracle transcription) and
tests/mgpu_triples_check.py (the (T) energy with units split over the ranks vs the oracle and vs one
rank) and tests/mgpu_next3_check.py (contract3 and sliced views with round-robin owners, gathered over
NCCL), one process per GPU over NCCL.  Skipped on boxes with fewer than 2 GPUs."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("script,marker,port", [("mgpu_check.py", "MGPU_CHECK PASS", 29531),
                                                ("mgpu_ccsd_check.py", "MGPU_CCSD_CHECK PASS", 29532),
                                                ("mgpu_triples_check.py", "MGPU_TRIPLES_CHECK PASS", 29533),
                                                ("mgpu_next3_check.py", "MGPU_NEXT3_CHECK PASS", 29534)])
def test_multigpu_script(script, marker, port):
    n = min(_ngpus(), 4)
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", script)]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert marker in out.stdout, out.stdout[-3000:]
