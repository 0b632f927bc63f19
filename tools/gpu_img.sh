# image-window kNN: parity tests, then the frame kNN-cov timing / fallback rate per window size, launch list, ncu
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q -k "knn or smoke or tracker or deterministic" -p no:cacheprovider > gpurun_out/pytest_img.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_img.log
for m in 6; do GSICP_IMG_M=$m timeout 300 python tools/img_diag.py > gpurun_out/img_diag_$m.txt 2>&1; echo diag$m rc=$?; cat gpurun_out/img_diag_$m.txt; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/img_frame_launches.csv python tools/knn_prof.py > /dev/null 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KREG:-k_knn_image}" -s 2 -c ${KC:-2} -o gpurun_out/prof_${NAME:-img} python tools/knn_prof.py > /dev/null 2>&1; echo ncu2 rc=$?
