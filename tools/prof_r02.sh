# profiling pass (two gpurun calls: the 64 MiB copy-back limit): PART=frame: launch list of the
# bench frame + ncu --set full (+ the SURVEY §8(d).4 metrics) of the frame's kernels + the k_align
# per-iteration timeline; PART=c4: the C4 map kNN (brick + warp search + grid) and the flat GN
# loop of an 8-frame batch, plus the C4 / batch timing tables.  TAG names the round / variant.
TAG=${TAG:-r02}
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -2
EXTRA="--metrics sm__inst_executed_pipe_fp64.sum,lts__t_bytes.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"
if [ "${PART:-frame}" = "frame" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --no-c4 --no-cpu-baseline --seq-frames 0 --batch 0 --no-configs > gpurun_out/${TAG}_launch_run.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full $EXTRA --clock-control none --import-source on -k regex:"k_align(<|$)|k_knn_image|k_knn_brute|k_align_seed|k_bp_" -s 20 -c 12 -o gpurun_out/${TAG}_frame python bench.py --steps 1 --warmup 3 --no-c4 --no-cpu-baseline --seq-frames 0 --batch 0 --no-configs > gpurun_out/${TAG}_frame_run.log 2>&1; echo ncu2 rc=$?
timeout 300 python tools/align_diag.py > gpurun_out/${TAG}_align_diag.txt 2>&1; echo diag rc=$?
python tools/align_iters_time.py > gpurun_out/${TAG}_align_iters.txt 2>&1
else
timeout 900 ncu --set full $EXTRA --clock-control none --import-source on -k regex:"k_knn_brick|k_knn_search|k_knn_epilogue|k_grid" -s 5 -c 6 -o gpurun_out/${TAG}_c4 python tools/c4_time.py 1 > gpurun_out/${TAG}_c4_run.log 2>&1; echo ncu3 rc=$?
timeout 900 ncu --set full $EXTRA --clock-control none --import-source on -k regex:"k_flat_" -s 0 -c 6 -o gpurun_out/${TAG}_batch python tools/batch_time.py 8 > gpurun_out/${TAG}_batch_run.log 2>&1; echo ncu4 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c4_launches.csv python tools/c4_time.py 1 > /dev/null 2>&1; echo ncu5 rc=$?
python tools/c4_time.py > gpurun_out/${TAG}_c4_time.txt 2>&1
python tools/batch_time.py 1,4,8,16 > gpurun_out/${TAG}_batch_time.txt 2>&1
python tools/c3_time.py > gpurun_out/${TAG}_c3_time.txt 2>&1
fi
ls -la gpurun_out
