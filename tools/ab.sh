#!/bin/bash
# usage: bash tools/ab.sh VARIANT...   (alternating bench runs of libfgc_b200.<v>.so; "cur" = the default lib)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = cur ]; then unset FGC_LIB_VARIANT; else export FGC_LIB_VARIANT=$v; fi
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stages_ms'].items() if not isinstance(x, str)})"
  done
done
