cd /root/repo
for cfg in 5 3; do for lib in default q0; do for sync in grid red; do
if [ "$lib" = default ]; then L=""; else L=paper_2012_03550_b200/lib/ab/$lib/libsgdt.so; fi
SGDT_LIB=$L SGDT_CORE_SYNC=$sync timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c$cfg $lib $sync', round(d['value']/1e9,2), 'core', round(d['phase_ms']['core'],4))"
done; done; done
