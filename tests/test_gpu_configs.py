"""Parity at BASELINE.json's hybrid configurations, through the fused
whole-step kernel, against the oracle replayed layer by layer
(decode_engine.hpp:109-151; tests/parity_util.py).

configs[1] Llama-3-8B 32K, top-k 2048, 32 layers, batch 1;
configs[2] Qwen3-8B 128K, top-k 4096, 36 layers, batch 1 -- the bench
           headline workload with bench.py's own role map (16 selection
           items per row, a layer with 3 retrieval heads);
configs[3] Llama-3-8B 64K, batch 16, top-k 512 and 8192 (1024 selection
           items of layer 0 over 144 CTAs);
configs[4] Llama-3-8B 256K, batch 4, top-k 2048, unsharded on one GPU
           (32 selection items per row).
The reduced-layer cases keep every distinct layer shape of the full model
(an all-retrieval layer 0, a 3-retrieval-head layer, single-retrieval and
all-sparse layers).  Each test prints and asserts the swap count (0, or
swaps inside the documented tie band).
"""
import json
import os

import numpy as np
import pytest
import torch

from tests.parity_util import roles_with, run_and_check

pytestmark = pytest.mark.gpu

H, G, D = 8, 4, 128
REDUCED = [(1, 0), (3, 1), (3, 4), (3, 6), (5, 2)]  # 6 layers: R at l1, 3 R at l3, R at l5


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_04541_b200  # noqa: F401
    torch.cuda.set_device(0)


def _report(name, rep):
    print(f"{name}: {rep}")
    out = os.environ.get("LYC_PARITY_REPORT")
    if out:
        with open(out, "a") as f:
            f.write(json.dumps({"config": name, **rep}) + "\n")


def test_llama3_8b_32k_all_layers(orc):
    import bench
    roles = bench.make_roles(32, H, 0.125, 2602)
    rep = run_and_check(orc, NL=32, B=1, H=H, G=G, d=D, L=32768, k=2048, roles=roles, seed=11)
    _report("llama3-8b-32k (32 layers, k 2048)", rep)


def test_qwen3_8b_128k_bench_config(orc):
    import bench
    roles = bench.make_roles(36, H, 0.125, 2602)
    assert (roles[1:] == 0).sum(1).max() >= 3  # the bench role map has a 3-retrieval layer
    rep = run_and_check(orc, NL=36, B=1, H=H, G=G, d=D, L=131072, k=4096, roles=roles, seed=12)
    _report("qwen3-8b-128k (36 layers, k 4096, bench roles)", rep)


@pytest.mark.parametrize("k", [512, 8192])
def test_llama3_8b_64k_batch16(orc, k):
    roles = roles_with(6, H, REDUCED)
    rep = run_and_check(orc, NL=6, B=16, H=H, G=G, d=D, L=65536, k=k, roles=roles, seed=13)
    _report(f"llama3-8b-64k b16 (6 layers, k {k})", rep)


def test_llama3_8b_256k_batch4(orc):
    roles = roles_with(6, H, REDUCED)
    rep = run_and_check(orc, NL=6, B=4, H=H, G=G, d=D, L=262144, k=2048, roles=roles, seed=14)
    _report("llama3-8b-256k b4 (6 layers, k 2048)", rep)
