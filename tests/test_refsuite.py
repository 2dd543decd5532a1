"""The reference's OWN GTest suites (proj/tests/test_solvers.cpp, test_recycle.cpp,
test_harness.cpp, test_precond.cpp), compiled unmodified by oracle/Makefile against a minimal GTest-compatible
header (oracle/gtest_mini):

* ref_<suite>  — linked with the reference library: pins gtest_mini (every assertion passes on the
  code the suites were written for);
* b200_<suite> — linked with the C++ drop-in shim (paper_1604_06043_b200/shim/idrstab_b200.cpp):
  every mstab::idrstab_solve / mstab_solve / sridr_solve the suites make, directly or through
  run_sequence (harness.cpp), runs on the B200 through libmstab_b200.so.

The binaries are built in the container that has /root/reference (build() / `make ref`) and travel
to the GPU box with the rest of oracle/_ref (git-ignored, not gpurun-ignored)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE_DIR = ROOT / "oracle" / "_ref" / "suite"
SUITES = ["test_solvers", "test_recycle", "test_harness", "test_precond"]


def run_suite(path):
    if not path.exists():
        pytest.fail(f"{path.relative_to(ROOT)} missing: run `make ref` where /root/reference exists")
    p = subprocess.run([str(path)], capture_output=True, text=True, timeout=900)
    ran = [ln for ln in p.stdout.splitlines() if ln.startswith("[ RUN")]
    failed = [ln for ln in p.stdout.splitlines() if ln.startswith("[  FAILED  ]")]
    assert p.returncode == 0 and not failed, (p.stdout[-4000:], p.stderr[-4000:])
    return len(ran)


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_reference(suite):
    """gtest_mini pinned: the suites pass against the reference library they were written for."""
    assert run_suite(SUITE_DIR / f"ref_{suite}") > 0


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200_shim(suite):
    """The reference's assertions hold with every solve routed through the B200 shim."""
    assert run_suite(SUITE_DIR / f"b200_{suite}") > 0


@pytest.mark.gpu
def test_complex_data_through_the_shim():
    """tests/shim/test_complex_shim.cpp: complex128 operators, right-hand sides and recycle data in
    the reference's own C++ types go through mstab::idrstab_solve / mstab_solve of the shim onto the
    B200 and are compared with the unmodified reference solve linked into the same binary."""
    assert run_suite(SUITE_DIR / "b200_test_complex_shim") == 3


@pytest.mark.gpu
def test_helper_cases_launch_kernels_through_the_shim():
    """The Arnoldi / BicgProjection / LevelIteration / PolyCombination cases of test_solvers.cpp run
    the shim's device-backed helpers: the library reports the kernels it launched at exit."""
    import os
    path = SUITE_DIR / "b200_test_solvers"
    if not path.exists():
        pytest.fail(f"{path.relative_to(ROOT)} missing: run `make ref` where /root/reference exists")
    env = dict(os.environ, MSTAB_REPORT_LAUNCHES="1")
    p = subprocess.run([str(path), "--gtest_filter=Arnoldi.*:BicgProjection.*:LevelIteration.*:PolyCombination.*"],
                       capture_output=True, text=True, timeout=600, env=env)
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    ran = [ln for ln in p.stdout.splitlines() if ln.startswith("[ RUN")]
    assert len(ran) >= 10, p.stdout[-2000:]
    line = [ln for ln in p.stderr.splitlines() if ln.startswith("[mstab] kernel launches:")]
    assert line and int(line[-1].split(":")[1]) > 100, p.stderr[-1000:]
