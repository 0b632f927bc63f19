# kNN-cov change check: build, the kNN / map / voxel / target parity tests, C4 timing + diag
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 -p no:cacheprovider -k "${PYTEST_K:-knn or map or voxel or target or wall}" > gpurun_out/pytest_knn.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_knn.log
python tools/c4_time.py 2>&1 | tee gpurun_out/c4_time.txt
python tools/c4_diag.py 2>&1 | tee gpurun_out/c4_diag.txt
