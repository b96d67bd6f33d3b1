"""Randomised parity sweep (scripts/fuzz_decode.py): random shapes, dtypes,
splits (including one split per batch item), roles and all four policies,
every case against the oracle's decode_step."""
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("seed,mode", [(3, ""), (11, ""), (5, "edge")])
def test_random_configs_match_oracle(seed, mode):
    """mode "edge": contexts of 1, 2, 63-65, 127 and 8191-8193 tokens, k >= seq,
    k = 1, odd group sizes."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, str(ROOT / "scripts" / "fuzz_decode.py"), str(seed), "12"] +
                       ([mode] if mode else []), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "bad cases: 0" in r.stdout, r.stdout[-3000:]
