"""Drop-in proof: the reference's own acceptance suite
(/root/reference/proj/tests/acceptance_main.cpp, SPEC criteria 1-10), compiled
unmodified against this repository's include/seqpipe headers and linked to
lib/libseqpipe_b200.so, with this repository's CLI (bin/seqpipe_b200) as
SEQPIPE_CLI_PATH (criterion 10 shells out to it).

The only addition is tests/acceptance/oracle_shim.*: the reference's test-only
exhaustive makespan oracle (validate.cpp:431-508) is out of scope here (SURVEY §2
row 9), so the shim declares it and throws; criterion 9 is therefore the one
expected failure. Everything else -- warm-up exactness, the 1F1B closed form,
bubble reduction, memory ordering, legality + 100 seeded mutations per kind,
partitioner quality, ablation and zero-bubble direction, byte determinism of the
CLI outputs -- must PASS.

CPU-only: needs the reference sources, so it runs in the build container and is
skipped where /root/reference is absent (the GPU box)."""
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = Path("/root/reference/proj/tests/acceptance_main.cpp")
LIB = ROOT / "paper_2406_03488_b200" / "lib" / "libseqpipe_b200.so"
CLI = ROOT / "paper_2406_03488_b200" / "bin" / "seqpipe_b200"


@pytest.mark.skipif(not SRC.exists(), reason="reference sources absent (GPU box)")
def test_reference_acceptance_suite_against_this_library(tmp_path):
    assert LIB.exists() and CLI.exists(), "run __graft_entry__.build() first"
    exe = tmp_path / "acceptance"
    shim = ROOT / "tests" / "acceptance"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", str(ROOT / "include"), "-I", str(shim),
                    "-include", str(shim / "oracle_shim.hpp"), f'-DSEQPIPE_CLI_PATH="{CLI}"',
                    str(SRC), str(shim / "oracle_shim.cpp"), "-o", str(exe), str(LIB),
                    f"-Wl,-rpath,{LIB.parent}"], check=True, capture_output=True, timeout=600)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    status = {int(m.group(2)): m.group(1) for m in re.finditer(r"^\[(PASS|FAIL)\]\s+(\d+)\.", r.stdout, re.M)}
    assert sorted(status) == list(range(1, 11)), r.stdout
    failed = sorted(c for c, s in status.items() if s == "FAIL")
    assert failed == [9], r.stdout  # only the out-of-scope exhaustive oracle
    assert "oracle_min_makespan is a test-only search" in r.stdout
