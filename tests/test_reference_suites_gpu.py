"""The reference's OWN unit tests (proj/tests/voxel_map_test.cpp, map_io_test.cpp,
search_test.cpp, angular_grid_test.cpp), compiled unmodified against the
B200 facade (include/bnbloc_b200.hpp) by tests/cpp/Makefile, run on the GPU.
Every map build, membership probe, score, batch_evaluate and search they
perform goes through libbbs_b200.so.  oracle_facade_test is our own
(tests/cpp/oracle_facade_test.cpp): harness_test.cpp's Oracle cases through
the facade's device-backed oracle_search."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "bin")


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["voxel_map_test", "search_test", "angular_grid_test",
                                   "map_io_test", "oracle_facade_test"])
def test_reference_suite_passes_on_device(suite):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (reference test sources absent when building)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    summary = [ln for ln in p.stdout.splitlines() if ln.startswith("[==========]")]
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    assert summary and summary[-1].endswith(" 0 failed"), summary
