# one gpurun call: GPU parity tests on the in-tree library, then an A/B over prebuilt variants
# (tools/build_variant.py; VARIANTS="a b ..." REPS=n as tools/gpu_abv.sh)
mkdir -p gpurun_out
cp paper_2403_12550_b200/libgsicp.so /tmp/libgsicp_intree.so
if [ -z "$NO_TESTS" ]; then
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -rf --timeout 600 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
fi
bash tools/gpu_abv.sh
cp /tmp/libgsicp_intree.so paper_2403_12550_b200/libgsicp.so
