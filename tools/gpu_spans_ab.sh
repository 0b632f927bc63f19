# frame stage spans (tools/frame_spans.py) per library variant, REPS rounds interleaved
L=paper_2403_12550_b200/libgsicp.so
cp $L /tmp/libgsicp_cur.so
for r in $(seq 1 ${REPS:-2}); do
for v in ${VARIANTS}; do
  cp paper_2403_12550_b200/variants/libgsicp_$v.so $L
  echo "$v $(python tools/frame_spans.py 2>&1 | tail -1)"
done
done
cp /tmp/libgsicp_cur.so $L
