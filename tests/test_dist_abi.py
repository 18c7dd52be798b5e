"""adi_create_dist: the in-library line-sharded handle with the NCCL
halo exchange inside adi_step.  Host logic here (CPU): the library's band plan equals
dist.band_partition (the plan the gloo / LocalGroup tests verify), and the NCCL unique
id is produced through the run-time-loaded libnccl.  The single-rank path runs in
tests/test_gpu_dist.py; multi-rank NCCL needs one GPU per rank (not available here)."""
import pytest

import paper_2006_07583_b200 as adi
from paper_2006_07583_b200 import dist


@pytest.mark.parametrize("npos,nranks", [(16384, 2), (16384, 4), (16384, 8), (2101, 3), (1601, 4),
                                          (517, 3), (301, 2), (1000, 7), (9, 1)])
def test_dist_bands_match_python_partition(npos, nranks):
    cuts = adi.adi_dist_bands(npos, nranks)
    bands = dist.band_partition(npos, nranks, 0)
    assert cuts == [a for a, _ in bands] + [bands[-1][1]]
    assert all((c - 1) % 4 == 0 for c in cuts[1:-1])   # 4-line groups for the row sweep


def test_nccl_unique_id():
    """In a subprocess: ncclGetUniqueId starts NCCL's bootstrap threads, and later tests
    fork (gloo ranks)."""
    import os
    import subprocess
    import sys
    code = ("import paper_2006_07583_b200 as a\n"
            "try:\n    u = a.adi_nccl_unique_id()\n"
            "except a.AdiError as e:\n    print('ENCCL' if e.code == a.ADI_ENCCL else 'ERR'); raise SystemExit\n"
            "print(len(u), int(any(u)))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=root,
                         timeout=120).stdout.strip()
    if out == "ENCCL":
        pytest.skip("libnccl not available")
    assert out == "128 1", out


def test_create_dist_argument_errors():
    with pytest.raises(adi.AdiError):
        adi.adi_create_dist(65, 65, 1 / 64, 0.5 / 64, 1.0, adi.ADI_MFD, 1, None, 0, 2)   # no id
    with pytest.raises(adi.AdiError):
        adi.adi_create_dist(65, 65, 1 / 64, 0.5 / 64, 1.0, adi.ADI_MFD, 1, b"\0" * 128, 2, 2)   # rank
    with pytest.raises(adi.AdiError):
        adi.adi_create_dist(65, 65, 1 / 64, 0.5 / 64, 1.0, adi.ADI_CFD_FULL, 1, b"\0" * 128, 0, 2)
