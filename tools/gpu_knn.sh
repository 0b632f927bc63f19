# kNN A/B: tile kernel (default) at a few qmin values vs the warp search of every point
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q -k "knn or smoke" -p no:cacheprovider > gpurun_out/pytest_knn.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_knn.log
for q in 30 12; do GSICP_TILE_QMIN=$q timeout 600 python tools/knn_diag.py > gpurun_out/knn_diag_tile$q.txt 2>&1; echo tile$q rc=$?; cat gpurun_out/knn_diag_tile$q.txt; done
GSICP_KNN=warp timeout 600 python tools/knn_diag.py > gpurun_out/knn_diag_warp.txt 2>&1; echo warp rc=$?; cat gpurun_out/knn_diag_warp.txt
