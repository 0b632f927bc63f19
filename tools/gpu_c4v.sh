# C4 A/B over prebuilt library variants (tools/build_variant.py): per variant the C4 timing
# (bench configuration first) and an ncu launch list of the same run.  VARIANTS="a b ..."
mkdir -p gpurun_out
L=paper_2403_12550_b200/libgsicp.so
cp $L /tmp/libgsicp_intree.so
for v in ${VARIANTS}; do
  cp paper_2403_12550_b200/variants/libgsicp_$v.so $L
  timeout 300 python tools/c4_time.py ${C4_CASES:-2} > gpurun_out/c4v_$v.txt 2>&1; echo "c4 $v rc=$?"
  cat gpurun_out/c4v_$v.txt
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4v_${v}_launches.csv python tools/c4_time.py 1 > /dev/null 2>&1; echo "ncu $v rc=$?"
  python tools/launch_table.py gpurun_out/c4v_${v}_launches.csv 2>&1 | head -14
done
cp /tmp/libgsicp_intree.so $L
