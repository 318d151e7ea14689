"""The multi-PROCESS engine data plane, executed on one GPU: P processes (rank r of world P,
one Engine each, all on cuda:0) exchange activations and gradients through the peer-memory
transport (transport_ipc.cu: CUDA-IPC-mapped receive rings + release / acquire flag words)
exactly as sp_comm_plan lists them -- the pipeline edges of the reference dependency model
(/root/reference/proj/core/src/sim.cpp:20-23 activations, :31-33 gradients). torch.distributed
(gloo) is only the side channel for the IPC blobs.

Checked per rank: the executed op log is the reference generate()'s device order; loss and every
parameter gradient match the fp64 oracle (relative L2 <= 1e-5 in the fp32 validation mode,
<= 2e-2 in the bf16 production mode)."""
import os
import pickle
import socket
import tempfile

import pytest

pytestmark = pytest.mark.gpu
TOL_F32 = 1e-5


def _model(E, GPT, world, bf16):
    if bf16:  # tcgen05 GEMMs + tensor-core attention at head dim 80
        return E.ModelConfig(family=GPT, dtype=E.BF16, vocab=512, hidden=320, layers=2 * world, heads=4, head_dim=80,
                             ffn=1280, max_seq=512, seed=42)
    return E.ModelConfig(family=GPT, dtype=E.F32, vocab=256, hidden=128, layers=2 * world, heads=2, head_dim=64,
                         ffn=256, max_seq=512, seed=42)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, k, out_dir, bf16=False):
    import torch.distributed as dist

    from oracle.transformer import GPT, tokens_for
    from paper_2406_03488_b200 import engine as E
    from paper_2406_03488_b200 import planner as pl

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    model = _model(E, GPT, world, bf16)
    cfg = pl.ScenarioConfig(pipeline_size=world, micro_batches=2 * world, segments=k, seq_len=512,
                            layers=model.layers, hidden_dim=model.hidden, param_count=model.param_count())
    part = pl.partition_for(cfg, "cwp" if k > 1 else "even")
    eng = E.Engine(cfg, kind, part, model, rank=rank, world_size=world, cuda_device=0)
    blob = eng.ipc_export()
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    eng.ipc_connect(blobs)
    tok = tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=5)
    rep = eng.step(tok)
    res = {"rank": rank, "loss": rep.loss, "order": eng.op_log().device_orders[rank],
           "params": {n: eng.read_param(n) for n in eng.params()},
           "grads": {n: eng.read_grad(n) for n in eng.params()}}
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,P,k,bf16", [("seq1f1b", 2, 4, False), ("seq1f1b", 4, 4, False), ("1f1b", 2, 1, False),
                                           ("seq1f1b", 2, 4, True)])
def test_multiprocess_ipc_step_matches_reference_order_and_oracle(gpu, kind, P, k, bf16):
    import torch.multiprocessing as mp

    from oracle import ref
    from oracle.transformer import GPT, Model, rel_l2, tokens_for
    from paper_2406_03488_b200 import planner as pl

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(P, _free_port(), kind, k, d, bf16), nprocs=P, join=True)
        res = []
        for r in range(P):
            with open(os.path.join(d, f"rank{r}.pkl"), "rb") as f:
                res.append(pickle.load(f))
    from paper_2406_03488_b200 import engine as E
    model = _model(E, GPT, P, bf16)
    tol = 2e-2 if bf16 else TOL_F32
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=2 * P, segments=k, seq_len=512, layers=model.layers,
                            hidden_dim=model.hidden, param_count=model.param_count())
    part = pl.partition_for(cfg, "cwp" if k > 1 else "even")
    want = ref.generate(cfg, kind, part).device_orders
    for r in range(P):
        assert res[r]["order"] == want[r], f"rank {r} executed a different order"
    params, grads_eng = {}, {}
    for x in res:
        params.update(x["params"])
        grads_eng.update(x["grads"])
    tok = tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=5)
    loss, grads = Model(GPT, model.vocab, model.hidden, model.layers, model.heads, model.head_dim,
                        model.ffn).step(params, tok, part.lengths)
    assert abs(res[P - 1]["loss"] - loss) / abs(loss) < tol, (res[P - 1]["loss"], loss)
    bad = {n: rel_l2(grads_eng[n], grads[n]) for n in params}
    assert max(bad.values()) < tol, bad


def _deadlock_worker(rank, world, port, out_dir):
    os.environ["SP_P2P_WATCHDOG_S"] = "5"  # read when the engine is created
    import time

    import torch.distributed as dist

    from oracle.transformer import GPT, tokens_for
    from paper_2406_03488_b200 import engine as E
    from paper_2406_03488_b200 import planner as pl

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    model = _model(E, GPT, world, False)
    cfg = pl.ScenarioConfig(pipeline_size=world, micro_batches=2 * world, segments=2, seq_len=512,
                            layers=model.layers, hidden_dim=model.hidden, param_count=model.param_count())
    eng = E.Engine(cfg, "seq1f1b", pl.partition_for(cfg, "cwp"), model, rank=rank, world_size=world, cuda_device=0)
    blobs = [None] * world
    dist.all_gather_object(blobs, eng.ipc_export())
    eng.ipc_connect(blobs)
    res = {"rank": rank}
    if rank == 0:  # rank 1 never steps: rank 0's first receive can never pair up
        t0 = time.time()
        try:
            eng.step(tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=5))
            res["error"] = None
        except pl.DeadlockError as e:
            res["error"] = str(e)
        res["seconds"] = time.time() - t0
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as f:
        pickle.dump(res, f)
    dist.barrier()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


def test_multiprocess_ipc_watchdog_turns_a_missing_peer_into_deadlock_error(gpu):
    """The reference's failure mode for a transfer that never pairs up (sim.cpp:217-231,
    DeadlockError) on the peer-memory transport: rank 1 never runs its step, rank 0's step
    raises DeadlockError after the watchdog (its parked stream waits are released) instead of
    hanging, and both processes tear down cleanly."""
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_deadlock_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        with open(os.path.join(d, "rank0.pkl"), "rb") as f:
            r0 = pickle.load(f)
    assert r0["error"] and "watchdog" in r0["error"], r0
    assert 4.0 < r0["seconds"] < 60.0, r0
