"""KV-sequence sharding as TWO real processes: each rank owns
its row slice of every head's cache in its own CUDA context and runs
ShardedDecoder -> lyc_shard_layer / lyc_shard_merge; the per-layer packed
exchange goes through an `exchange` callback over a gloo process group
(device -> host -> all_gather -> device; the NCCL all-gather's CPU-staged
stand-in, since this pool gives one GPU per call).  Both ranks must produce
bitwise identical outputs and global index sets, equal to the oracle's
decode_step (decode_engine.hpp:109-151) within the north_star tolerances,
sets exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.test_gpu_decode import BF16_TOL, FP32_TOL, rel_err, roles_for, synth

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_exchange(send: torch.Tensor, recv: torch.Tensor):
    """all_gather of every rank's packed block in rank order, staged on the host."""
    torch.cuda.current_stream().synchronize()
    host = send.cpu()
    parts = [torch.empty_like(host) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, host)
    recv.copy_(torch.cat(parts).to(recv.device))


def _rank(rank, world, port, cfg, outdir):
    import paper_2602_04541_b200 as P
    from paper_2602_04541_b200.sharded import ShardedDecoder, shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    NL, B, H, G, d, seq, k, dtype, seed, roles = (cfg[x] for x in (
        "NL", "B", "H", "G", "d", "seq", "k", "dtype", "seed", "roles"))
    q, K, V = synth(seed, NL, B, H, G, d, seq, seq, dtype)
    rb, nl = shard_rows(seq, world, rank)
    Kl = K[..., rb:rb + nl, :].contiguous().cuda()  # this rank's rows only
    Vl = V[..., rb:rb + nl, :].contiguous().cuda()
    sd = ShardedDecoder(n_layers=NL, batch=B, n_kv_heads=H, group_size=G, d_head=d,
                        seq_cap=nl, roles=roles, policy=P.SparsityPolicy.top_k(k), dtype=dtype,
                        world=world, rank=rank, exchange=_gloo_exchange)
    gsets = torch.full((NL, B * H, sd.k_cap), -7, dtype=torch.int32, device="cuda")
    out = sd.decode_step(q.cuda(), Kl, Vl, nl, rb, seq, global_sets=gsets)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), out=out.float().cpu().numpy(),
             sets=gsets.cpu().numpy())
    sd.close()
    dist.barrier()
    dist.destroy_process_group()


def _last_retrieval(roles, g):
    return max(l for l in range(roles.shape[0]) if l == 0 or roles[l, g] == 0)


@pytest.mark.parametrize("case", ["tiny_fp32", "llama_bf16"])
def test_two_process_sequence_shards_vs_oracle(orc, tmp_path, case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if case == "tiny_fp32":
        cfg = dict(NL=4, B=1, H=2, G=4, d=64, seq=4096, k=256, dtype=torch.float32, seed=5,
                   roles=roles_for(4, 2, [(2, 1)]))
        tol = FP32_TOL
    else:
        cfg = dict(NL=3, B=2, H=8, G=4, d=128, seq=16384, k=1024, dtype=torch.bfloat16, seed=9,
                   roles=roles_for(3, 8, [(1, 3), (2, 5), (2, 0)]))
        tol = BF16_TOL
    world = 2
    mp.start_processes(_rank, args=(world, _free_port(), cfg, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    assert np.array_equal(res[0]["out"], res[1]["out"]), "ranks disagree on the output"
    assert np.array_equal(res[0]["sets"], res[1]["sets"]), "ranks disagree on the global sets"
    NL, B, H, G, d, seq, k, roles = (cfg[x] for x in ("NL", "B", "H", "G", "d", "seq", "k", "roles"))
    q, K, V = synth(cfg["seed"], NL, B, H, G, d, seq, seq, cfg["dtype"])
    for b in range(B):
        ref = orc.decode_step(q[:, b].float().numpy(), K[:, b].float().numpy(),
                              V[:, b].float().numpy(), roles, seq=seq, scale=1 / np.sqrt(d),
                              kind="topk", k=k)
        err = rel_err(res[0]["out"][:, b], ref["out"])
        assert err < tol, (b, err)
        for g in range(H):
            l = _last_retrieval(roles, g)
            np.testing.assert_array_equal(res[0]["sets"][l, b * H + g, :k], ref["sets"][g])
