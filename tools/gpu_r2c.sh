#!/bin/bash
# Round-2: full GPU suite + benches of every workload (+ guard-mode suite).
T=${1:-r2c}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${T}_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/${T}_pytest_gpu.log
for wl in c1 c2 c3 c5; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_$wl.json 2> gpurun_out/${T}_bench_$wl.err; echo "bench $wl rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${T}_bench_$wl.json'));print('$wl',round(d['value']),round(d['ms_per_step'],3),'K3',round(d['roofline']['frac'],3),d['stage_ms'])"
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo "bench c4 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${T}_bench_c4.json'));print('c4',round(d['value']),round(d['ms_per_step'],3),'K3',round(d['roofline']['frac'],3),d['stage_ms'],'e2e',round(d['e2e']['value']))"
if [ "${GUARD:-1}" = "1" ]; then
BSM_GUARD=1 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu_guard.log 2>&1; echo "guard pytest rc=$?"
tail -4 gpurun_out/${T}_pytest_gpu_guard.log
fi
