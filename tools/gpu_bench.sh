set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/ncu_launch_run.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_align$|k_knn_search|k_knn_epilogue|k_grid_" -s 2 -c 4 -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/ncu_full_run.log 2>&1; echo ncu2 rc=$?
tail -5 gpurun_out/ncu_full_run.log
ls -la gpurun_out
