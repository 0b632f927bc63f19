mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
CUDA_LAUNCH_BLOCKING=1 timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke_dbg.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke_dbg.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke_memcheck.log 2>&1; echo memcheck rc=$?
head -80 gpurun_out/smoke_memcheck.log
