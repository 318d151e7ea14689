"""Diagnose the multi-process peer-memory transport on one GPU: P processes, progress printed
per phase with timestamps, a traceback dump if a phase stalls. Usage:
  SP_P2P_WATCHDOG_S=30 python tools/ipc_debug.py [--P 2] [--k 4] [--kind seq1f1b] [--bf16]"""
import argparse
import faulthandler
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def log(rank, msg):
    print(f"[{time.time() % 1000:8.3f}] rank {rank}: {msg}", file=sys.stderr, flush=True)


def gdb_dump(rank):
    import subprocess
    out = os.path.join("gpurun_out", f"ipcdbg_gdb_rank{rank}.txt")
    with open(out, "w") as f:
        subprocess.run(["timeout", "60", "cuda-gdb", "-p", str(os.getpid()), "-batch", "-ex", "thread apply all bt 25",
                        "-ex", "info cuda kernels"], stdout=f, stderr=subprocess.STDOUT)
    log(rank, f"gdb dump -> {out}")


def worker(rank, world, port, kind, k, bf16, steps, idle_rank=-1):
    import threading
    faulthandler.dump_traceback_later(150, exit=True)
    t = threading.Timer(float(os.environ.get("IPC_DBG_GDB_S", "45")), gdb_dump, args=(rank,))
    t.daemon = True
    t.start()
    import torch.distributed as dist

    from oracle.transformer import GPT, tokens_for
    from paper_2406_03488_b200 import engine as E
    from paper_2406_03488_b200 import planner as pl

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    log(rank, "gloo up")
    if bf16:
        model = E.ModelConfig(family=GPT, dtype=E.BF16, vocab=512, hidden=320, layers=2 * world, heads=4,
                              head_dim=80, ffn=1280, max_seq=512, seed=42)
    else:
        model = E.ModelConfig(family=GPT, dtype=E.F32, vocab=256, hidden=128, layers=2 * world, heads=2,
                              head_dim=64, ffn=256, max_seq=512, seed=42)
    cfg = pl.ScenarioConfig(pipeline_size=world, micro_batches=2 * world, segments=k, seq_len=512,
                            layers=model.layers, hidden_dim=model.hidden, param_count=model.param_count())
    part = pl.partition_for(cfg, "cwp" if k > 1 else "even")
    eng = E.Engine(cfg, kind, part, model, rank=rank, world_size=world, cuda_device=0)
    log(rank, "engine built")
    blob = eng.ipc_export()
    log(rank, f"exported {len(blob)} B")
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    eng.ipc_connect(blobs)
    log(rank, "connected")
    dist.barrier()
    tok = tokens_for(cfg.micro_batches, cfg.seq_len, model.vocab, seed=5)
    if rank == idle_rank:  # never steps: the peers' transfers with this rank cannot pair up
        log(rank, "idle (not stepping)")
        steps = 0
    for i in range(steps):
        t0 = time.time()
        try:
            rep = eng.step(tok)
            log(rank, f"step {i}: loss {rep.loss:.6f} in {time.time() - t0:.3f} s")
        except Exception as e:  # noqa: BLE001
            log(rank, f"step {i} FAILED after {time.time() - t0:.1f} s: {type(e).__name__}: {e}")
            if idle_rank < 0:
                os._exit(3)
            break
    log(rank, "closing")
    eng.close()
    log(rank, "closed")
    t.cancel()
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--kind", default="seq1f1b")
    ap.add_argument("--bf16", action="store_true")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--idle-rank", type=int, default=-1, help="this rank never steps (watchdog check)")
    a = ap.parse_args()
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(worker, args=(a.P, port, a.kind, a.k, a.bf16, a.steps, a.idle_rank), nprocs=a.P, join=True)
    print("ok", file=sys.stderr)


if __name__ == "__main__":
    main()
