set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 600 python tools/align_diag.py > gpurun_out/align_diag.txt 2>&1; echo adiag rc=$?
cat gpurun_out/align_diag.txt
timeout 600 python tools/knn_diag.py > gpurun_out/knn_diag.txt 2>&1; echo diag rc=$?
cat gpurun_out/knn_diag.txt
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-c4 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
