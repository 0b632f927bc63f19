# frame-batch timing over library variants (VARIANTS="a b"): tools/batch_time.py per variant
L=paper_2403_12550_b200/libgsicp.so
cp $L /tmp/libgsicp_cur.so
for v in ${VARIANTS}; do
  cp paper_2403_12550_b200/variants/libgsicp_$v.so $L
  echo "== $v"; python tools/batch_time.py ${BS:-1,2,4,8,16} 2>&1 | tail -5
done
cp /tmp/libgsicp_cur.so $L
