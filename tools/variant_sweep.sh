#!/bin/bash
# Time attention fwd/bwd for each library variant: tools/variant_sweep.sh v1 v2 ...
for v in base "$@"; do
  for shape in "6674 26094 32 80" "10170 0 32 80" "8192 8192 32 128"; do
    if [ "$v" = base ]; then r=$(python tools/attn_once.py $shape); else r=$(python tools/attn_once.py --variant $v $shape); fi
    echo "$v [$shape]: $r"
  done
done
