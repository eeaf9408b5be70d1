#!/bin/bash
# BASELINE.json configs 3 and 4 on one box: AlexNet-sized (61M floats) keep
# ratio sweep and VGG-16-sized (138M floats) range-float width sweep, one
# bench.py line each (N from $1, default 1), into gpurun_out/sweeps_n$N.jsonl.
N=${1:-1}
mkdir -p gpurun_out
OUT=gpurun_out/sweeps_n$N.jsonl
: > $OUT
CPU=""
[ "$N" != "1" ] && CPU="--no-cpu-baseline"
for t in 0.99 0.95 0.9 0.7; do
  timeout 600 python bench.py --gpus $N --workload alexnet --theta-drop $t --steps 10 --warmup 3 $CPU 2>>gpurun_out/sweeps_n$N.err | tail -1 >> $OUT
done
for nb in 4 6 8 16; do
  timeout 600 python bench.py --gpus $N --workload vgg16 --n-bits $nb --steps 10 --warmup 3 $CPU 2>>gpurun_out/sweeps_n$N.err | tail -1 >> $OUT
done
python - "$OUT" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    try:
        d = json.loads(l)
    except ValueError:
        print("bad line:", l[:200]); continue
    c = d["config"]
    print(f'{c["n"]:>10} theta_drop={c["theta_drop"]:<5} ({c["n_bits"]},{c["mantissa_bits"]}) N={d["n_gpus"]} '
          f'{d["ms_per_step"]:.3f} ms {d["value"]:.0f} GB/s ratio {d["compression_ratio"]:.1f} '
          f'frac {d["roofline"]["frac"]:.3f} e2e {d["e2e"]["value"]:.1f} GB/s '
          f'allreduce {d.get("allreduce_fp32_ms")} cpu {d.get("cpu_baseline", {}).get("value")}')
PY
