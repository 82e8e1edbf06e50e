#!/usr/bin/env bash
# A/B of a factor-kernel switch on BASELINE configs: ENV="VAR" VALS="0 1" CFGS="3"
cd "$(dirname "$0")/.."
OUT=gpurun_out/factor_ab
mkdir -p $OUT
for cfg in ${CFGS:-3}; do
  for v in ${VALS:-0 1}; do
    env $ENV=$v timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e \
      > $OUT/c${cfg}_${ENV}_$v.json 2>/dev/null
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']/1e9,2), [round(x,3) for x in d['phase_ms']['factor_modes']])" $OUT/c${cfg}_${ENV}_$v.json
  done
done
