"""Host side of the multi-process tensor-parallel wiring, on CPU with gloo
(world size 2): the IPC-handle exchange every rank runs before its first
pass, and the shard-shape validation of the C ABI."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_02493_b200 import espec as E


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = bytes([rank + 1]) * 64
    got = E.exchange_ipc_handles(mine)
    q.put((rank, got))
    dist.barrier()
    dist.destroy_process_group()


def test_ipc_handle_exchange_gloo_world2():
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([r + 1]) * 64 for r in range(world)]
    assert res[0] == want and res[1] == want


def test_exchange_rejects_bad_handle():
    with pytest.raises(ValueError):
        E.exchange_ipc_handles(b"short")


@pytest.mark.parametrize("tp,n_heads,d_mlp,vocab", [(3, 4, 128, 258), (2, 4, 48, 258), (4, 4, 128, 258), (9, 4, 128, 258)])
def test_tp_shard_shape_validation(tp, n_heads, d_mlp, vocab):
    base = E.ModelConfig(vocab_size=vocab, d_model=64, n_layers=4, n_heads=n_heads, d_head=16, d_mlp=d_mlp,
                         max_positions=128)
    with pytest.raises(E.EspecError) as ei:
        E.Engine(base, base, E.RunConfig(n=4, lp_size=2), tp_size=tp, tp_rank=0)
    assert ei.value.kind == "config"
