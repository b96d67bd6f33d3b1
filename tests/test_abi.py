"""CPU checks of the product library: it loads, exports every symbol the public
header declares, and its host-side planner / cost model agree with the oracle
(no kernel launches here -- there is no GPU in this container)."""
import re

import numpy as np
import pytest

from tests.conftest import ROOT


def header_symbols():
    text = (ROOT / "include" / "lyc.h").read_text()
    return sorted(set(re.findall(r"\b(lyc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2602_04541_b200 import _lib
    L = _lib.lib()
    declared = header_symbols()
    assert declared, "no symbols parsed from include/lyc.h"
    for s in declared:
        assert hasattr(L, s), f"liblyc.so does not export {s}"
    assert sorted(_lib.SYMBOLS) == declared
    assert L.lyc_version().startswith(b"lyc-b200")


def test_plan_splits_matches_oracle(orc, golden):
    from paper_2602_04541_b200 import BlockIndexSet, plan_splits
    g = golden["plan_splits"]
    n = len([k for k in g if k.startswith("units")])
    for i in range(n):
        hb = g[f"hb{i}"]
        B, H = hb.shape
        bis = BlockIndexSet(B, H, [list(range(hb[b, h])) for b in range(B) for h in range(H)])
        s = plan_splits(bis, int(g[f"S{i}"]))
        assert s.split_blocks == g[f"sb{i}"].tolist()
        assert s.head_split_count == g[f"hsc{i}"].tolist()
        rec = [(b, si, u.kv_head, u.begin, u.end, u.head_local_split)
               for b in range(B) for si in range(s.num_splits) for u in s.units[b][si]]
        assert rec == [tuple(r) for r in g[f"units{i}"].tolist()]


def test_plan_splits_errors():
    from paper_2602_04541_b200 import BlockIndexSet, InvalidArgument, plan_splits
    with pytest.raises(InvalidArgument):
        plan_splits(BlockIndexSet(1, 2, [[], []]), 2)
    with pytest.raises(InvalidArgument):
        plan_splits(BlockIndexSet(1, 1, [[0, 1, 2, 3]]), 0)


def test_latency_model_matches_oracle(orc):
    from paper_2602_04541_b200 import BlockIndexSet, latency_model, plan_splits
    rng = np.random.default_rng(48)
    for rep in range(100):
        heads = int(rng.integers(2, 9))
        hb = rng.integers(1, 65, size=(1, heads))
        bis = BlockIndexSet(1, heads, [list(range(x)) for x in hb[0]])
        c = latency_model(plan_splits(bis, heads), 64)
        o = orc.latency_model(hb, heads, 64)
        assert c.pooled_critical_blocks == o["pooled_critical_blocks"]
        assert c.naive_critical_blocks == o["naive_critical_blocks"]
        assert c.balance_ratio == o["balance_ratio"]
        assert c.pooled_critical_blocks <= c.naive_critical_blocks  # kernel_sim_test.cpp:294-315


def test_fraction_budget_matches_oracle(orc):
    from paper_2602_04541_b200 import fraction_budget
    for n in (1, 2, 7, 100, 4096, 131072):
        for f in (1e-9, 0.1, 0.3, 0.5, 0.7, 0.999):
            assert fraction_budget(f, n) == orc.fraction_budget(f, n)


def test_gemv_validates_before_launch():
    """lyc_gemv (toy_model.hpp:161-274 ops) rejects bad descriptors on the host
    with LYC_EINVAL / LYC_ENOTSUP -- no device needed."""
    import ctypes as C

    from paper_2602_04541_b200 import _lib as LL
    L = LL.lib()

    def rc(**kw):
        base = dict(M=64, K=64, w=0x1000, x=0x2000, xb=None, gain=None, eps=0.0,
                    mode=LL.GEMV_STORE, y=0x3000)
        base.update(kw)
        return L.lyc_gemv(C.byref(LL.lyc_gemv_desc(**base)), None)

    assert rc(w=None) == -1                       # null weights
    assert rc(K=60) == -1                         # K not a multiple of 8
    assert rc(K=50000) == -4                      # the input vector exceeds shared memory
    assert rc(xb=0x4000) == -1                    # both inputs
    assert rc(x=None) == -1                       # no input
    assert rc(w=0x1008) == -1                     # misaligned weights
    assert rc(x=0x2004) == -1                     # misaligned input vector
    assert rc(gain=0x2008) == -1                  # misaligned rmsnorm gain
    assert rc(prefetch=0x8004, prefetch_bytes=4096) == -1  # misaligned prefetch hint
    assert rc(flags=2) == -1                      # unknown flag
    assert rc(mode=9) == -1                       # unknown epilogue
    assert rc(mode=LL.GEMV_STORE, y=None) == -1
    assert rc(mode=LL.GEMV_SILU_BF16, y=None) == -1
    # QKV_ROPE: M must be (nq + 2 nkv) d, d even
    assert rc(mode=LL.GEMV_QKV_ROPE, q_out=0x5000, k_cache=0x6000, v_cache=0x7000,
              nq=2, nkv=1, d=16, M=63) == -1
    assert rc(mode=LL.GEMV_QKV_ROPE, q_out=0x5000, k_cache=0x6000, v_cache=0x7000,
              nq=2, nkv=1, d=15, M=60) == -1
    assert b"gemv" in L.lyc_last_error()


def test_decoder_entry_points_validate_before_launch():
    """refresh / sync on a null decoder, bad layers and lengths: host errors."""
    from paper_2602_04541_b200 import _lib as LL
    L = LL.lib()
    assert L.lyc_decoder_refresh_sets(None, 0, None, None, 1, None) == -1
    assert L.lyc_decoder_sync_sets(None, None) == -1
    assert L.lyc_decoder_tune(None, LL.TUNE_DEFER_SELECTION, 0) == -1
