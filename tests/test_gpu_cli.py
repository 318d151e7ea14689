"""`seqpipe_b200 execute`: the CLI runs the generated op table on the B200 and
writes the MEASURED step as seqpipe.simreport.v1 (+ timeline). The executed
task order per device must be the reference generate() order (oracle/_ref)."""
import json
import subprocess
from pathlib import Path

import pytest

from oracle import ref

pytestmark = pytest.mark.gpu
CLI = Path(__file__).resolve().parent.parent / "paper_2406_03488_b200" / "bin" / "seqpipe_b200"


@pytest.fixture(scope="module", autouse=True)
def _cli_built():
    if not CLI.exists():  # snapshot without the binary: link it against the shipped library (g++ only)
        from paper_2406_03488_b200 import build as B
        B._build_cli(verbose=False)
    assert CLI.exists()

TINY = """pipeline_size = 4
stages_per_device = 1
micro_batches = 6
segments = 4
seq_len = 1024
layers = 8
hidden_dim = 256
param_count = 6291456
cost_model = flops
"""


@pytest.mark.parametrize("kind,dtype,family", [("seq1f1b", "bf16", "gpt"), ("seqzb1p", "f32", "gpt"),
                                               ("seq1f1b", "bf16", "llama")])
def test_execute_writes_measured_report(tmp_path, gpu, kind, dtype, family):
    cfgf = tmp_path / "tiny.cfg"
    cfgf.write_text(TINY)
    heads = "4" if family == "gpt" else "2"
    r = subprocess.run([str(CLI), "execute", "--config", str(cfgf), "--kind", kind, "--partition", "cwp",
                        "--family", family, "--heads", heads, "--vocab", "512", "--ffn", "1024", "--dtype", dtype,
                        "--steps", "2",
                        "--out", str(tmp_path / "rep.json"), "--gantt", "ascii", "--gantt-width", "80", "--summary"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    doc = json.loads((tmp_path / "rep.json").read_text())
    assert doc["schema"] == "seqpipe.simreport.v1" and doc["kind"] == kind
    cfg = ref.parse_scenario_text(TINY)
    part = ref.partition_for(cfg, "cwp")
    assert doc["partition"] == part.lengths
    want = ref.generate(cfg, kind, part)
    for dev, order in zip(doc["devices"], want.device_orders):
        assert [(t["kind"], t["m"], t["s"]) for t in dev["tasks"]] == [(t.kind, t.micro_batch, t.segment) for t in order]
    rows = r.stdout.splitlines()
    assert rows[0].startswith(f"kind={kind} makespan=") and len(rows) == 5
    assert "tokens_per_s=" in r.stderr and "loss=" in r.stderr
