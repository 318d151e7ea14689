#!/usr/bin/env bash
# TEST INFRASTRUCTURE: compiles the UNMODIFIED reference seqpipe core from the
# sources where they lie (/root/reference/proj/core/src, read-only) plus our C
# shim into oracle/_ref/libseqpipe_ref.so. Nothing is copied into the repo; the
# reference's own CMake is not used (it needs the absent vendor/ tree). Its
# only third-party dependency is nlohmann/json (json_io.cpp:6), satisfied by
# the nlohmann 3.11.3 header shipped inside this image's cudnn_frontend wheel.
# The .so is git-ignored but travels to the GPU box with the snapshot.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${SEQPIPE_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
NLOHMANN="${NLOHMANN_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
if [ ! -d "$REF/core/src" ]; then
  echo "reference sources not present ($REF); using prebuilt $OUT if any" >&2
  exit 0
fi
mkdir -p "$OUT/obj"
# System g++ (same toolchain and libstdc++ as the engine build); ignores a CXX that may
# point at a toolchain linking its own static libstdc++.
CXX="${REF_CXX:-/usr/bin/g++}"
# The reference defines the same seqpipe:: C++ symbols as the engine library; a
# version script (ref_exports.map) keeps them local to this .so so a process
# that loads both can never bind one library's calls to the other's code.
FLAGS=(-std=c++20 -O2 -fPIC -I"$REF/core/include" -I"$NLOHMANN" -I"$HERE/../include")
pids=()
for src in "$REF"/core/src/*.cpp "$HERE/ref_shim.cpp"; do
  obj="$OUT/obj/$(basename "${src%.cpp}").o"
  if [ ! -f "$obj" ] || [ "$src" -nt "$obj" ]; then
    "$CXX" "${FLAGS[@]}" -c "$src" -o "$obj" &
    pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
"$CXX" -shared -Wl,--version-script="$HERE/ref_exports.map" -o "$OUT/libseqpipe_ref.so" "$OUT"/obj/*.o
echo "$OUT/libseqpipe_ref.so"
