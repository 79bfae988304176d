import pathlib
import subprocess
import sys

import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size) test")
    # CPU-side native pieces (generator + oracle) are cheap to build; build them if absent.
    need = [ROOT / "stencil_inputs" / "libstinputs.so", ROOT / "oracle" / "liboracle.so"]
    if not all(p.exists() for p in need):
        subprocess.run(["make", "-C", str(ROOT), "cpu"], check=True, capture_output=True)


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_lib():
    """The product library; on a GPU box it MUST load (no fallback)."""
    if not gpu_available():
        pytest.skip("no CUDA device")
    import paper_2310_01882_b200 as st
    st.lib()  # raises if libstencil.so is missing
    return st
