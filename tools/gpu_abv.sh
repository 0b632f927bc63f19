# A/B over prebuilt library variants (tools/build_variant.py): VARIANTS="base pf0 ..." ; each is
# copied over the in-tree libgsicp.so before a bench run; REPS repetitions interleaved
mkdir -p gpurun_out
L=paper_2403_12550_b200/libgsicp.so
for r in $(seq 1 ${REPS:-2}); do
for v in ${VARIANTS}; do
  cp paper_2403_12550_b200/variants/libgsicp_$v.so $L
  timeout 600 python bench.py --steps 30 --warmup 5 ${BENCH_ARGS:---no-cpu-baseline --no-c4 --batch 0 --seq-frames 60} > gpurun_out/abv_$v.json 2> gpurun_out/abv_$v.err; echo "bench $v rc=$?"
  python -c "
import json; d=json.load(open('gpurun_out/abv_$v.json'))
print('$v', 'value', round(d['value'],1), 'k_align', round(d['kernel_ms']['k_align']*1e3,1), 'p50', round(d['ms_p10_p50_p90'][1]*1e3,1), 'seq', round(d.get('sequence',{}).get('aligns_per_s',0),1), 'c3s4', d.get('c3_s4',{}).get('ms_p10_p50_p90',[0,0])[1], 'c3s1', d.get('c3_s1',{}).get('ms_p10_p50_p90',[0,0])[1])"
done
done
