"""Multi-process pipeline path on CPU: world_size 2 and 4 over torch.distributed
gloo. Each rank executes exactly the P2P plan the multi-process engine issues
(sp_comm_plan, derived from the op table), with NCCL's semantics emulated:
sends are asynchronous, receives block, and every (peer, channel) pair is a
FIFO. Each message carries its (kind, micro-batch, segment, stage) header; the
receiver checks it against what its own plan expects, and a toy per-stage map
(x -> 2x + stage) checks that activations and gradients compose end to end.
A deadlock (plans that do not pair up) fails the test through the timeout."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, P, M, k, kind, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_03488_b200 import engine as E
    from paper_2406_03488_b200 import planner as pl
    cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=k, seq_len=8 * k, cost_model="uniform")
    part = pl.even_partition(cfg) if kind != "seq1f1b" else pl.cwp_partition(
        pl.ScenarioConfig(**{**cfg.__dict__, "cost_model": "flops", "layers": 2, "hidden_dim": 4}))
    hidden = 2
    plan = E.comm_plan(cfg, kind, part, rank + 1, hidden)
    order = pl.generate(cfg, kind, part).device_orders[rank]
    by_op = {}
    for c in plan:
        by_op.setdefault((c["op_index"], c["when"]), []).append(c)
    acts = {}   # (m, s) -> activation tensor this stage produced
    pending = []
    V = P
    ok = True
    for j, t in enumerate(order):
        key = (t.micro_batch, t.segment)
        recv = None
        for c in by_op.get((j, "pre"), []):
            buf = torch.zeros(4 + c["elems"])
            # FIFO per (peer, channel): gloo tag = channel
            dist.recv(buf, src=c["peer"], tag=c["channel"])
            hdr = tuple(int(x) for x in buf[:4])
            want = ({"F": 0, "B": 1}[c["task"][0]], c["task"][1], c["task"][2], c["task"][3])
            ok &= hdr == want
            recv = buf[4:]
        n = part.lengths[t.segment - 1] * hidden
        if t.kind == "F":
            x = recv if recv is not None else torch.full((n,), float(t.micro_batch * 10 + t.segment))
            y = 2 * x + t.stage
            acts[key] = y
            out = y
        else:
            g = recv if recv is not None else torch.ones(n) * t.stage
            out = 2 * g  # d(2x + c)/dx = 2
        for c in by_op.get((j, "post"), []):
            hdr = torch.tensor([{"F": 0, "B": 1}[t.kind], t.micro_batch, t.segment, c["task"][3] + (1 if t.kind == "F"
                                                                                                    else -1)],
                               dtype=torch.float32)
            pending.append(dist.isend(torch.cat([hdr, out]), dst=c["peer"], tag=c["channel"]))
        if t.kind == "F" and t.stage == V:
            results[("last", key)] = float(out[0])
        if t.kind == "B" and t.stage == 1:
            results[("first_grad", key)] = float(out[0])
    for p in pending:
        p.wait()
    results[("ok", rank)] = ok
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("P,M,k,kind", [(2, 4, 2, "seq1f1b"), (2, 3, 1, "1f1b"), (4, 8, 4, "seq1f1b"),
                                        (4, 5, 3, "gpipe")])
def test_p2p_plan_pairs_across_ranks(P, M, k, kind):
    with mp.Manager() as man:
        results = man.dict()
        port = _free_port()
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_worker, args=(r, P, port, P, M, k, kind, results)) for r in range(P)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=120)
        alive = [p for p in procs if p.is_alive()]
        for p in alive:
            p.kill()
        assert not alive, "P2P plan deadlocked"
        assert all(p.exitcode == 0 for p in procs)
        res = dict(results)
    assert all(res[("ok", r)] for r in range(P))
    for m in range(1, M + 1):
        for s in range(1, k + 1):
            x = float(m * 10 + s)
            for v in range(1, P + 1):
                x = 2 * x + v
            assert res[("last", (m, s))] == x          # activations composed through every stage
            assert res[("first_grad", (m, s))] == P * 2 ** P  # gradient 2 per stage, seeded with P at the last
