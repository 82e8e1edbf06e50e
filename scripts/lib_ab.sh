#!/usr/bin/env bash
# A/B of library variants (scripts/build_variant.py) on BASELINE configs:
# VARIANTS="default s0g0 ..." CFGS="3 2" STEPS=5 bash scripts/lib_ab.sh
cd "$(dirname "$0")/.."
OUT=gpurun_out/lib_ab
mkdir -p $OUT
for cfg in ${CFGS:-3}; do
  for v in ${VARIANTS:-default}; do
    if [ "$v" = default ]; then lib=""; else lib=paper_2012_03550_b200/lib/ab/$v/libsgdt.so; fi
    SGDT_LIB=$lib timeout 900 python bench.py --config $cfg --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e \
      > $OUT/c${cfg}_$v.json 2>$OUT/c${cfg}_$v.err
    python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value']/1e9,2), [round(x,3) for x in d['phase_ms']['factor_modes']], round(d['phase_ms']['core'],3))" $OUT/c${cfg}_$v.json
  done
done
