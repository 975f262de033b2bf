# A/B of the pixels per k_mask_q CTA (BSM_MASKQ_PX): parity suite at the candidate, then per-stage times
mkdir -p gpurun_out
A=${1:-16}; B=${2:-32}
BSM_MASKQ_PX=$B timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab_pytest$B.log 2>&1; echo pytest$B rc=$?; tail -1 gpurun_out/ab_pytest$B.log
for wl in c4 c1 c5; do for px in $A $B $A $B; do
  BSM_MASKQ_PX=$px timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${wl}_$px.json 2>/dev/null
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab_${wl}_$px.json').read().strip().splitlines()[-1]);print('$wl px=$px',round(d['value']),d['stage_ms'])"
done; done
