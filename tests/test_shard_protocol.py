"""The sequence-sharding protocol over a real 2-process gloo
group on CPU: each rank computes its local split-KV partial and local top-k
candidates with the ORACLE on its row slice, one packed all-gather exchanges
them, and the rank-ordered LSE merge + global top-k over the gathered
candidates reproduce the unsharded oracle exactly (sets) / to 1e-12 (f64
outputs).  This pins the algebra the device path (lyc_shard_layer /
lyc_shard_merge) implements; no device code runs here."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, K, V, k, result):
    from oracle import pyoracle
    from paper_2602_04541_b200.sharded import shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = pyoracle.orc()
    L, d = K.shape
    rb, nl = shard_rows(L, world, rank)
    scale = 1 / np.sqrt(d)
    Ks, Vs = K[rb:rb + nl], V[rb:rb + nl]
    out, w = orc.dense_attention(q, Ks, Vs, scale)
    s = Ks.astype(np.float64) @ q.astype(np.float64) * scale
    m = s.max()
    lse = np.log(np.exp(s - m).sum()) + m
    loc = orc.args_top_k(s, k)                       # local top-k (ascending)
    cand = np.full((k, 2), -np.inf)
    cand[:len(loc), 0] = s[loc]
    cand[:len(loc), 1] = loc + rb
    block = torch.tensor(np.concatenate([out, [lse], cand.ravel()]), dtype=torch.float64)
    gathered = [torch.empty_like(block) for _ in range(world)]
    dist.all_gather(gathered, block)
    g = torch.stack(gathered).numpy()
    o_all, lse_all, c_all = g[:, :d], g[:, d], g[:, d + 1:].reshape(world, k, 2)
    M = lse_all.max()
    wts = np.exp(lse_all - M)
    merged = (wts[:, None] * o_all).sum(0) / wts.sum()
    cands = c_all.reshape(-1, 2)                     # rank order = ascending global id
    order = np.lexsort((cands[:, 1], -cands[:, 0]))  # key desc, id asc
    glob = np.sort(cands[order[:k], 1].astype(np.int64))
    result[rank] = (merged, glob)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_protocol_matches_unsharded_oracle(world):
    from oracle import pyoracle
    rng = np.random.default_rng(5)
    L, d, k = 1500, 32, 64
    q = rng.uniform(-1, 1, d)
    K = rng.uniform(-1, 1, (L, d))
    V = rng.uniform(-1, 1, (L, d))
    mgr = mp.Manager()
    result = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, q, K, V, k, result), nprocs=world, join=True)
    orc = pyoracle.orc()
    ref_out, w = orc.dense_attention(q, K, V, 1 / np.sqrt(d))
    ref_set = orc.args_top_k(w, k)
    for r in range(world):
        merged, glob = result[r]
        np.testing.assert_allclose(merged, ref_out, rtol=0, atol=1e-12)
        np.testing.assert_array_equal(glob, ref_set)
    np.testing.assert_array_equal(result[0][0], result[1][0])  # identical on every rank


def test_shard_rows_partition():
    from paper_2602_04541_b200.sharded import shard_rows
    for L in (1, 7, 4096, 262144):
        for P in (1, 2, 3, 8):
            spans = [shard_rows(L, P, p) for p in range(P)]
            assert spans[0][0] == 0
            for (b0, n0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + n0 == b1
            assert sum(n for _, n in spans) == L
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
