# align change check: build, the align / GN / batch / LM / sequence parity tests, then the A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as e; e.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -q -x -rf --timeout 600 -p no:cacheprovider -k "${PYTEST_K:-align or gn or iteration or batch or lm or sequence or c3 or linearize or pose or map or keyframe}" > gpurun_out/pytest_align.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_align.log
cp paper_2403_12550_b200/libgsicp.so /tmp/libgsicp_cur.so
VARIANTS="${VARIANTS}" REPS=${REPS:-2} bash tools/gpu_abv.sh
cp /tmp/libgsicp_cur.so paper_2403_12550_b200/libgsicp.so
