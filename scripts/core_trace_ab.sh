#!/usr/bin/env bash
# Core-phase A/B with the CTA-0 cycle trace: SYNCS="grid red" GRIDS="148 64" CFG=2
cd "$(dirname "$0")/.."
for sync in ${SYNCS:-grid red}; do for g in ${GRIDS:-148}; do
echo "== sync $sync grid $g"
SGDT_CORE_TRACE=1 SGDT_CORE_SYNC=$sync SGDT_CORE_GRID=$g timeout 600 python bench.py --config ${CFG:-2} --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2> gpurun_out/trace_c${CFG:-2}_${sync}_$g.err | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e9,2), 'core', round(d['phase_ms']['core'],4))"
grep "core trace" gpurun_out/trace_c${CFG:-2}_${sync}_$g.err | tail -1
done; done
