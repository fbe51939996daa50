import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def rel_err(got, ref):
    """Per-tensor parity metric of SURVEY.md §8: (max|d|/max|ref|, ||d||/||ref||)."""
    got = np.asarray(got, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    d = got - ref
    mref = np.abs(ref).max() if ref.size else 0.0
    nref = np.linalg.norm(ref)
    rmax = np.abs(d).max() / mref if mref > 0 else np.abs(d).max() if d.size else 0.0
    rl2 = np.linalg.norm(d) / nref if nref > 0 else np.linalg.norm(d)
    return float(rmax), float(rl2)


TOL = 1e-4  # fp32 GPU vs fp64 oracle, per tensor (north_star "within 1e-4 relative")


def assert_close(got, ref, tol=TOL, what=""):
    rmax, rl2 = rel_err(got, ref)
    assert rmax <= tol and rl2 <= tol, f"{what}: max-rel {rmax:.3e}, l2-rel {rl2:.3e} > {tol:g}"


@pytest.fixture(scope="session")
def oracle_port():
    from oracle import port
    return port()


@pytest.fixture(scope="session")
def oracle_ref():
    from oracle import ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return ref()


@pytest.fixture(scope="module")
def pk():
    import paper_2505_22208_b200 as pk
    return pk


@pytest.fixture(scope="module")
def dev(pk):
    import cases
    d = pk.Device(pk.ModelConfig(*cases.CFG[:3], cutoff=cases.CFG[3], heads=cases.CFG[4]), seed=7)
    d.set_option("export_fp64", 1)
    yield d
    d.close()
