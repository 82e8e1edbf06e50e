#!/usr/bin/env bash
# A/B of an environment switch on BASELINE configs: ENV="VAR" VALS="a b" CFGS="2 3" STEPS=10
# prints value (G updates/s), the per-mode factor times and the core time.
cd "$(dirname "$0")/.."
OUT=gpurun_out/env_ab
mkdir -p $OUT
for cfg in ${CFGS:-3}; do
  for v in ${VALS:-0 1}; do
    env $ENV=$v timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e \
      > $OUT/c${cfg}_${ENV}_$v.json 2>$OUT/c${cfg}_${ENV}_$v.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']/1e9,2), [round(x,3) for x in d['phase_ms']['factor_modes']], 'core', round(d['phase_ms']['core'],4))" $OUT/c${cfg}_${ENV}_$v.json
  done
done
