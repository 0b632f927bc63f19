set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 600 python tools/align_diag.py > gpurun_out/align_diag.txt 2>&1; echo adiag rc=$?
cat gpurun_out/align_diag.txt
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-c4 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_align$|k_knn_search" -s 2 -c 2 -o gpurun_out/prof_$NCU python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/ncu_full_run.log 2>&1; echo ncu2 rc=$?
fi
