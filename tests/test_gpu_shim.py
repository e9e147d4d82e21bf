"""INTEGRATION.md §2's C++ shim run on the GPU: acr::GpuFactorization::make / solve through the
C-ABI from a C++ program (poisson n=8 residual), and the error mapping of the singular case
to acr::SingularBlockError(level 0, plane 2) (test_acr.cpp:223-241)."""
import subprocess

import pytest

from test_boundary import build_shim

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return build_shim(str(tmp_path_factory.mktemp("shim") / "acr_shim_check"))


def test_cpp_shim_factor_solve(exe):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("shim ok")


def test_cpp_shim_singular_error(exe):
    r = subprocess.run([exe, "singular"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "level 0 plane 2" in r.stdout
