# one gpurun call: build, GPU tests, bench, optional diagnostics (DIAG="align overlap knn")
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(round(d['value'],1), d['stage_ms_eager'], d['kernel_ms'], d.get('knn_cov_4M_ms'), round(d['e2e']['value'],1))"
tail -3 gpurun_out/bench.err
for d in ${DIAG}; do timeout 600 python tools/${d}_diag.py > gpurun_out/${d}_diag.txt 2>&1; echo $d rc=$?; head -${DIAG_LINES:-40} gpurun_out/${d}_diag.txt; done
