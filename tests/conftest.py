import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def pytest_terminal_summary(terminalreporter):
    """Per-config parity table (max-abs / max-rel vs the fp64 oracle, beside SDPA-bf16's error) at
    the end of every run that executed GPU parity cases — so the driver's GPU test log carries it."""
    mod = sys.modules.get("test_gpu_parity") or sys.modules.get("tests.test_gpu_parity")
    rows = getattr(mod, "RESULTS", None)
    if not rows:
        return
    tr = terminalreporter
    tr.section("parity vs the fp64 CPU oracle (BASELINE.md §4)")
    tr.write_line(f"{'case':62s} {'max_abs':>9s} {'max_rel':>9s} {'sdpa_bf16':>9s} {'>quantum':>9s} bound")
    for name, a, r, b, q, bound in rows:
        tr.write_line(f"{name[:62]:62s} {a:9.3e} {r:9.3e} {b:9.3e} {q:9.3e} {bound}")
