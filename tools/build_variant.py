#!/usr/bin/env python
"""Build a tuning variant of the product library with extra nvcc defines for one
CUDA source: tools/build_variant.py NAME SOURCE.cu -DFOO=1 ...  ->
paper_2406_03488_b200/lib/variants/libseqpipe_b200_NAME.so. Used only for kernel
tuning sweeps on the GPU box: a tool loads it by pointing _capi.LIB_PATH at it
before the first _capi.lib() call (tools/attn_once.py --variant NAME); the
product loader honours no environment switch."""
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2406_03488_b200 import build as B  # noqa: E402

name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
B.build()
out = B.OUT / "variants"
out.mkdir(exist_ok=True)
srcp = B.CSRC / "cuda" / src
obj = out / f"{src}.{name}.o"
subprocess.run([B.NVCC, *B.NVFLAGS, *B.INCLUDES, *defs, "-c", str(srcp), "-o", str(obj)], check=True)
objs = [p for p in sorted(B.OBJ.glob("*.o")) if not p.name.startswith("cuda__" + src)] + [obj]
lib = out / f"libseqpipe_b200_{name}.so"
subprocess.run([B.NVCC, "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                *map(str, objs), "-o", str(lib), f"-L{B.CUDA / 'lib64'}", "-lcudart", *B.NCCL_LINK, "-ldl",
                "-Xlinker", "-rpath,$ORIGIN/.."], check=True)
print(lib)
