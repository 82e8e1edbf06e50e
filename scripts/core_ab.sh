#!/usr/bin/env bash
# A/B of the core-phase paths on BASELINE configs (phase_ms.core from bench.py):
# the cooperative column kernel vs the blocked steps at several block widths.
cd "$(dirname "$0")/.."
OUT=gpurun_out/core_ab
mkdir -p $OUT
run() {  # cfg mode T steps
  SGDT_CORE=$2 SGDT_CORE_T=$3 timeout 600 python bench.py --config $1 --steps $4 --warmup 3 --no-cpu-baseline --no-e2e \
    > $OUT/c$1_$2_T$3.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']/1e9,2), round(d['phase_ms']['core'],4))" $OUT/c$1_$2_T$3.json
}
for cfg in ${CFGS:-2 3}; do
  run $cfg column 0 10
  for T in ${TS:-0 2 5 10}; do run $cfg blocked $T 10; done
done
