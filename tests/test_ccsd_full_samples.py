"""Full-size parity of the configs[3] CCSD iteration (O=100, V=800, tile 50, N_L=1800, alpha/beta maps):
sampled R1 / R2 elements that tools/bench_ccsd.py --samples-out read from the GPU run (committed under
profiles/), rechecked on the host by oracle/ccsd_sample.py -- the element-wise form of the literal
oracle, pinned to it on mini shapes (tests/test_ccsd_iteration.py) -- from the seeded input recipe
alone.  Bar: normwise 1e-11 (reading R13; the norm is the largest |reference| over the samples, a
lower bound of max |R|).  Runs with different GPU counts must agree bit for bit (R12: every tensor
element is computed whole by one rank)."""
import glob
import json
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = sorted(glob.glob(os.path.join(ROOT, "profiles", "r02_ccsd_samples_n*.json")))


@pytest.mark.skipif(not FILES, reason="no committed sample files")
def test_gpu_counts_agree_bitwise():
    recs = [json.load(open(f)) for f in FILES]
    for r in recs[1:]:
        assert r["r2"] == recs[0]["r2"] and r["r1"] == recs[0]["r1"], "sampled elements differ across GPU counts"


@pytest.mark.skipif(not FILES, reason="no committed sample files")
def test_recorded_host_check():
    """Every committed run carries the full host recheck of all its samples (done on the GPU box)."""
    for f in FILES:
        r = json.load(open(f))
        assert r["check"]["r2_normwise"] <= 1e-11 and r["check"]["r1_normwise"] <= 1e-11, f


@pytest.mark.skipif(not FILES, reason="no committed sample files")
def test_resample_subset_on_host():
    """Recompute two R2 and two R1 samples of the first file here (about a minute of host BLAS)."""
    from oracle.ccsd_sample import Inputs, Sampler
    r = json.load(open(FILES[0]))
    c = r["config"]
    sm = Sampler(Inputs(c["O"], c["V"], c["N_L"], c["seed"]))
    ref2 = np.array(r["check"]["r2_ref"])
    norm2, norm1 = np.abs(ref2).max(), np.abs(np.array(r["check"]["r1_ref"])).max()
    for (a, b, i, j, g) in r["r2"][:2]:
        assert abs(sm.r2(a, b, i, j) - g) <= 1e-11 * norm2, (a, b, i, j)
    for (a, i, g) in r["r1"][:2]:
        assert abs(sm.r1(a, i) - g) <= 1e-11 * norm1, (a, i)
