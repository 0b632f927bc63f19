# C4 profiling pass: per-kernel launch list of the 4e6-point kNN-cov, brick diagnostics,
# ncu --set full of the brick kernel and the warp-search leftovers.  TAG names the variant.
TAG=${TAG:-c4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -2
python tools/c4_time.py > gpurun_out/${TAG}_time.txt 2>&1
python tools/c4_diag.py > gpurun_out/${TAG}_diag.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/c4_time.py 1 > /dev/null 2>&1; echo ncu1 rc=$?
EXTRA="--metrics sm__inst_executed_pipe_fp64.sum,lts__t_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"
timeout 900 ncu --set full $EXTRA --clock-control none --import-source on -k regex:"k_knn_brick|k_knn_search|k_grid_insert|k_knn_epilogue" -s 8 -c 5 -o gpurun_out/${TAG}_full python tools/c4_time.py 1 > gpurun_out/${TAG}_ncu_run.log 2>&1; echo ncu2 rc=$?
cat gpurun_out/${TAG}_time.txt gpurun_out/${TAG}_diag.txt
