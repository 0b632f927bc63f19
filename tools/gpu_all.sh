# one gpurun call: build, GPU parity tests, bench, ncu launch list + full capture of the hot kernels
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 400 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -n "$NCU" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-c4 --no-cpu-baseline --seq-frames 0 --batch 0 > gpurun_out/ncu_launch_run.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_align(<|$)|k_knn_image|k_knn_brute|k_align_seed" -s 5 -c 10 -o gpurun_out/prof_$NCU python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline --seq-frames 0 --batch 0 > gpurun_out/ncu_full_run.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_align_batch" -s 1 -c 1 -o gpurun_out/prof_${NCU}_batch python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline --seq-frames 0 --batch 4 > gpurun_out/ncu_batch_run.log 2>&1; echo ncu3 rc=$?
fi
