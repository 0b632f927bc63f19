set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 600 python tools/align_diag.py > gpurun_out/align_diag.txt 2>&1; echo rc=$?; cat gpurun_out/align_diag.txt
