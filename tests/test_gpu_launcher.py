"""GPU-resident launcher core: the device cwp partition and the device op
tables are bit-identical to the compiled reference (oracle/_ref)."""
import itertools

import pytest

from oracle import ref
from paper_2406_03488_b200 import planner as pl

pytestmark = pytest.mark.gpu


def _cfgs():
    for name in ("gpt-2.7b", "gpt-7b", "gpt-13b", "gpt-30b"):
        yield pl.preset_scenario(name)
    base = pl.preset_scenario("gpt-2.7b")
    for P, T, k in [(4, 32768, 4), (8, 65536, 8), (8, 131072, 16), (8, 16384, 2)]:
        c = pl.preset_scenario("gpt-13b" if T == 131072 else "gpt-7b" if T == 65536 else "gpt-2.7b")
        c.pipeline_size, c.seq_len, c.segments = P, T, k
        yield c
    for n, k, L, d, p in itertools.product([100, 513, 2048, 4097], [2, 3, 5, 8], [1, 8], [8, 256], [0, 1000, 6291456]):
        if n >= k:
            yield pl.ScenarioConfig(pipeline_size=2, micro_batches=4, segments=k, seq_len=n, layers=L, hidden_dim=d,
                                    param_count=p)


def test_device_cwp_bit_exact(gpu):
    n = 0
    for cfg in _cfgs():
        assert pl.device_partition(cfg, "cwp") == ref.partition_for(cfg, "cwp").lengths, cfg
        assert pl.device_partition(cfg, "even") == ref.partition_for(cfg, "even").lengths
        n += 1
    assert n > 100


@pytest.mark.parametrize("kind", ["gpipe", "1f1b", "seq1f1b"])
def test_device_op_tables_bit_exact(gpu, kind):
    for P, M, k in itertools.product([1, 2, 3, 4, 8], [1, 2, 4, 5, 8, 9, 16, 32], [1, 2, 3, 4, 8, 16]):
        cfg = pl.ScenarioConfig(pipeline_size=P, micro_batches=M, segments=k, seq_len=16 * k, cost_model="uniform")
        part = pl.partition_for(cfg, "even")
        assert pl.device_schedule(cfg, kind).device_orders == ref.generate(cfg, kind, part).device_orders, (P, M, k)


def test_device_op_table_rejects_interleaved(gpu):
    cfg = pl.ScenarioConfig(pipeline_size=2, stages_per_device=2, micro_batches=4, segments=2, seq_len=32)
    with pytest.raises(pl.UnsupportedScheduleError):
        pl.device_schedule(cfg, "seq1f1b-i")
