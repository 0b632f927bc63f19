# one gpurun call: build, GPU parity tests, then bench A/B over an env switch (AB_VAR=name, AB_VALS="a b")
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
for v in ${AB_VALS}; do
  env ${AB_VAR}=$v timeout 600 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; echo bench $v rc=$?
  python -c "import json,sys; d=json.load(open('gpurun_out/bench_$v.json')); print('$v', round(d['value'],1), d['stage_ms_eager'], d['kernel_ms'], d.get('knn_cov_4M_ms'), round(d['e2e']['value'],1))"
  tail -3 gpurun_out/bench_$v.err
done
