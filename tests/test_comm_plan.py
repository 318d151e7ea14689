"""The P2P plan the multi-rank engine executes (sp_comm_plan), checked on CPU over a grid of
every schedule kind: one channel per pipeline edge and direction, exactly one sending and one
receiving device per channel, and the receiver posts exactly the sender's messages in the
sender's order -- so per-channel FIFOs (NCCL communicator + stream per channel) pair up by
construction, for interleaved schedules too (where two stage edges join the same device pair).
The engine runs the same check (comm_plan_check) before it launches anything."""
import itertools

import pytest

from paper_2406_03488_b200 import engine as E
from paper_2406_03488_b200 import planner as pl

KINDS = ["gpipe", "1f1b", "seq1f1b", "1f1b-i", "seq1f1b-i", "zb1p", "seqzb1p"]


def _cfg(P, nv, M, k):
    return pl.ScenarioConfig(pipeline_size=P, stages_per_device=nv, micro_batches=M, segments=k, seq_len=16 * k,
                             layers=2 * P * nv, hidden_dim=8, param_count=1000)


def _tag(c):
    kind, m, s, stage = c["task"]
    if c["dir"] == "send":
        return (kind in ("B", "I"), m, s, stage)
    return (kind in ("B", "I"), m, s, stage - 1 if kind == "F" else stage + 1)


@pytest.mark.parametrize("kind", KINDS)
def test_every_channel_pairs_fifo_by_construction(kind):
    checked = 0
    for P, nv, M, k in itertools.product([2, 3, 4], [1, 2, 3], [2, 3, 4, 6, 8], [1, 2, 3, 4]):
        if pl.is_interleaved(kind) != (nv > 1):
            continue
        cfg = _cfg(P, nv, M, k)
        try:
            part = pl.even_partition(cfg)
            sched = pl.generate(cfg, kind, part)
        except pl.InvalidArgument:  # infeasible point (reference feasibility rules)
            continue
        V = P * nv
        senders, receivers = {}, {}
        for d in range(1, P + 1):
            for c in E.comm_plan(cfg, kind, part, d, 8):
                side = senders if c["dir"] == "send" else receivers
                side.setdefault(c["channel"], {"dev": set(), "seq": []})
                side[c["channel"]]["dev"].add(d)
                side[c["channel"]]["seq"].append((_tag(c), c["elems"]))
        assert set(senders) == set(receivers)
        assert all(0 <= ch < 2 * (V - 1) for ch in senders)
        for ch in senders:
            assert len(senders[ch]["dev"]) == 1 and len(receivers[ch]["dev"]) == 1, (P, nv, M, k, ch)
            assert senders[ch]["seq"] == receivers[ch]["seq"], (kind, P, nv, M, k, ch)
        assert len(senders) == (2 * (V - 1) if P > 1 else 0) or nv > 1 or P == 1
        checked += 1
        del sched
    assert checked > 0
