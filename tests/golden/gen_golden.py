#!/usr/bin/env python
"""Generates tests/golden/planner_golden.json from the UNMODIFIED reference
planner (oracle/_ref/libseqpipe_ref.so, built by oracle/build_ref.sh from
/root/reference/proj/core/src). Run in the build container (the reference is
not present on the GPU box); the JSON is committed so the tests can pin the
engine's planner against reference outputs anywhere.

    python tests/golden/gen_golden.py
"""
import json
import sys
from fractions import Fraction
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_2406_03488_b200 import planner as pl  # noqa: E402


def frac(x: Fraction) -> str:
    return f"{x.numerator}/{x.denominator}"


def cfg_dict(c: pl.ScenarioConfig) -> dict:
    d = {}
    for k, v in c.__dict__.items():
        d[k] = frac(v) if isinstance(v, Fraction) else v
    return d


def scenarios():
    out = {}
    # cfg-T: tiny GPT, param_count = exact trainable count of the engine's tiny model (V=512, T=2048)
    tiny = pl.ScenarioConfig(pipeline_size=4, micro_batches=8, segments=4, seq_len=2048, layers=8, hidden_dim=256,
                             param_count=8 * (2 * 256 + 4 * 256 * 256 + 2 * 256 * 1024) + 2 * 512 * 256 + 2048 * 256 + 256)
    out["cfgT_tiny_gpt"] = tiny
    out["cfgT_survey_12Ld2"] = pl.ScenarioConfig(pipeline_size=4, micro_batches=8, segments=4, seq_len=2048, layers=8,
                                                hidden_dim=256, param_count=12 * 8 * 256 * 256)
    for name, preset, P, T, k, M in [("cfg2_gpt2.7b_32k", "gpt-2.7b", 4, 32768, 4, 8),
                                     ("cfg3_7b_64k", "gpt-7b", 8, 65536, 8, 16),
                                     ("cfg4_13b_128k", "gpt-13b", 8, 131072, 16, 16),
                                     ("bench_p1_gpt2.7b_32k", "gpt-2.7b", 1, 32768, 4, 8)]:
        c = ref.preset_scenario(preset)
        for key, val in (("pipeline_size", P), ("seq_len", T), ("segments", k), ("micro_batches", M)):
            c = ref.apply_scenario_override(c, key, str(val))
        out[name] = c
    out["sample_cfg"] = ref.parse_scenario_text((Path("/root/reference/proj/configs/sample.cfg")).read_text())
    return out


def main():
    gold = {"generator": "oracle/_ref (reference seqpipe core) via tests/golden/gen_golden.py", "scenarios": {}}
    for name, cfg in scenarios().items():
        entry = {"config": cfg_dict(cfg), "partitions": {}, "schedules": {}, "simulate": {}}
        for mode in ("even", "cwp"):
            p = ref.partition_for(cfg, mode)
            entry["partitions"][mode] = {"lengths": p.lengths, "imbalance": frac(p.imbalance)}
        p = ref.partition_for(cfg, "cwp")
        for kind in ("1f1b", "seq1f1b", "gpipe"):
            c = cfg
            if kind == "1f1b":
                c = pl.ScenarioConfig(**{**cfg.__dict__, "segments": 1})
                pk = ref.partition_for(c, "even")
            else:
                pk = p
            s = ref.generate(c, kind, pk)
            entry["schedules"][kind] = [" ".join(f"{t.kind}{t.micro_batch}.{t.segment}" for t in o)
                                        for o in s.device_orders]
            timings, devs, summ, n = ref.simulate_raw(s, pk)
            entry["simulate"][kind] = {
                "makespan": frac(pl._frac(summ.makespan)),
                "aggregate_bubble_ratio": frac(pl._frac(summ.aggregate_bubble_ratio)),
                "max_peak_memory": frac(pl._frac(summ.max_peak_memory)),
                "modeled_throughput": frac(pl._frac(summ.modeled_throughput)),
                "peak_allocations": [devs[d].peak_allocations for d in range(c.pipeline_size)],
                "bubble_ratio": [frac(pl._frac(devs[d].bubble_ratio)) for d in range(c.pipeline_size)],
            }
        gold["scenarios"][name] = entry
    out = Path(__file__).with_name("planner_golden.json")
    out.write_text(json.dumps(gold, indent=1))
    print(out, out.stat().st_size)


if __name__ == "__main__":
    main()
