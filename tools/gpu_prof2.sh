# ncu of one script's kernels: SCRIPT=tools/x.py KREGEX=... NAME=...
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${NAME}_launches.csv python ${SCRIPT} > /dev/null 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${SKIP:-0} -c ${COUNT:-2} -o gpurun_out/prof_${NAME} python ${SCRIPT} > gpurun_out/ncu_${NAME}.log 2>&1; echo ncu2 rc=$?
grep -E "k_align_seed|k_knn" gpurun_out/${NAME}_launches.csv | tail -8
