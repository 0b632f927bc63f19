# one gpurun call: build, GPU parity tests (all, failures listed), smoke, bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -3 gpurun_out/smoke.log
if [ -n "$PYTEST_K" ]; then
timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
else
timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
fi
tail -30 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
fi
