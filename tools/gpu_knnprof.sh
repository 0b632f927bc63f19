# launch lists (device time per kernel) of the kNN-cov path on the bench frame and on C4, plus one
# full ncu capture of the tile kernel on the bench frame
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${NAME}_frame_launches.csv python tools/knn_prof.py > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${NAME}_c4_launches.csv python tools/knn_prof.py c4 > /dev/null 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_knn_tile}" -s ${SKIP:-1} -c 1 -o gpurun_out/prof_${NAME} python tools/knn_prof.py > gpurun_out/ncu_${NAME}.log 2>&1; echo ncu3 rc=$?
