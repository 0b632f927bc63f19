# ncu --set full of the C4 brick kernel only (one launch), source-correlated. TAG names the variant.
TAG=${TAG:-brick}
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_knn_brick" -s 2 -c 1 -o gpurun_out/${TAG} python tools/c4_time.py 1 > gpurun_out/${TAG}_run.log 2>&1; echo ncu rc=$?
python tools/c4_time.py 1
