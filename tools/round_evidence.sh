mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_v19.log 2>&1; echo "rc smoke $?"
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_v19.log 2>&1; echo "rc pytest $?"; tail -1 gpurun_out/pytest_gpu_v19.log
for wl in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v19_$wl.jsonl 2>gpurun_out/bench_$wl.err; echo "rc bench $wl $?"; done
timeout 900 python bench.py > gpurun_out/bench_v19_cfg2.jsonl 2>gpurun_out/bench_cfg2.err; echo "rc bench cfg2 $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_v19_reference_arm.jsonl 2>gpurun_out/bench_ref.err; echo "rc ref $?"
for f in gpurun_out/bench_v19_*.jsonl; do python -c "import json,sys;d=json.loads(open('$f').readlines()[-1]);print('$f',d.get('config',{}).get('workload'),'%.3e'%d['value'],'e2e %.3e'%d['e2e']['value'],d.get('clocks',{}).get('reasons'))"; done
