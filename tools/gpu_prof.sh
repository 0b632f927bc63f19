set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KERN" -s ${SKIP:-2} -c 1 -o gpurun_out/prof_$NCU python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/ncu_full_run.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_full_run.log
