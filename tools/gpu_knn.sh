set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
for v in warp thread; do GSICP_KNN=$v timeout 600 python tools/knn_diag.py > gpurun_out/knn_diag_$v.txt 2>&1; echo $v rc=$?; cat gpurun_out/knn_diag_$v.txt; done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_knn_thread" -s 2 -c 1 -o gpurun_out/prof_$NCU python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline > gpurun_out/ncu_full_run.log 2>&1; echo ncu2 rc=$?
fi
