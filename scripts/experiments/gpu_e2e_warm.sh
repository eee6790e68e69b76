# e2e after warming every distinct step's pinned buffers (default bench, twice)
python -m paper_2605_08962_b200.build > gpurun_out/build.log 2>&1 || exit 1
for r in 1 2; do
  MUX_E2E_TRACE=1 python bench.py > gpurun_out/ew_$r.json 2> gpurun_out/ew_$r.err
  grep "e2e trace" gpurun_out/ew_$r.err | head -1 | cut -c1-1500
  python -c "
import json;d=json.loads(open('gpurun_out/ew_$r.json').read().strip().splitlines()[-1])
print('cfg2', round(d['value']/1e6,2), d['e2e']['variants'])
print('t1', round(d['target1']['value']/1e6,2), d['target1']['e2e']['variants'])"
done
