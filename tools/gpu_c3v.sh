# C3 timing over library variants (VARIANTS="a b"): tools/c3_time.py with each variant swapped in
L=paper_2403_12550_b200/libgsicp.so
cp $L /tmp/libgsicp_cur.so
for v in ${VARIANTS}; do
  cp paper_2403_12550_b200/variants/libgsicp_$v.so $L
  echo "== $v"; python tools/c3_time.py 2>&1 | tail -3 | cut -c1-80
done
cp /tmp/libgsicp_cur.so $L
