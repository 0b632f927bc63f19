set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/smoke.log
tail -40 gpurun_out/pytest_gpu.log
