"""The multi-process tensor-parallel wiring on one B200: two processes (one
per TP rank, as torchrun would start on two GPUs) export their receive
regions as CUDA IPC handles, all-gather them over a gloo process group and
run the single-kernel collectives (push over mapped peer memory, release/
acquire flags at system scope). Both ranks share cuda:0 here, so the GPU
time-slices the two contexts; the tokens must still equal the reference
fixture."""
import json
import os
import socket
from dataclasses import replace

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_generate.json")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, idx, q, layout="tp"):
    import torch.distributed as dist

    from paper_2502_02493_b200 import espec as E
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = json.load(open(GOLDEN))[idx]
        r = case["run"]
        base = E.ModelConfig(**{k: case["base"][k] for k in ("vocab_size", "d_model", "n_layers", "n_heads", "d_head",
                                                            "d_mlp", "max_positions", "norm_eps", "seed")})
        run = E.RunConfig(algorithm=r["algorithm"], n=r["n"], widths=r["widths"], lp_size=r["lp_size"],
                          plan_override=r["plan_override"] or None, temperature=r["temperature"],
                          max_new_tokens=min(r["max_new_tokens"], 24), seed=r["seed"], calibration=r["calibration"])
        eng = E.Engine(base, replace(base, n_layers=case["keep"]), run, device=0, tp_size=world, tp_rank=rank,
                       draft_layout=layout)
        eng.link_process_group()
        eng.init_weights(E.Engine.BASE, base.seed)
        if layout == "tp":
            eng.share_truncated_draft()
        else:  # the layer-parallel drafter: init_model(keep layers, same seed)
            eng.init_weights(E.Engine.DRAFT, base.seed)
        toks, _ = eng.generate(case["prompt"].encode())
        q.put((rank, [int(t) for t in toks], case["tokens"][:len(toks)]))
        eng.close()
    except Exception as ex:  # reported to the parent
        q.put((rank, repr(ex), None))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("layout", ["tp", "lp"])
def test_tp2_two_processes_ipc_matches_reference(layout):
    world, port = 2, _port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, port, 3, q, layout)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, got, want in res:
        assert want is not None, got
        assert got == want
