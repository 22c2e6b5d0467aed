mkdir -p gpurun_out
for v in base minb base minb; do
  cp gpurun_lib_$v.so paper_2201_04265_b200/libldpc_b200.so
  for c in T1-R1/4:1000 T1-R1/2:1000 T1-R1/4:100000 T1-R1/2:100000; do
    cfg=${c%%:*}; fr=${c##*:}
    echo "== $v $cfg $fr" >> gpurun_out/minb_ab.log
    timeout 200 python bench.py --config $cfg --frames $fr --no-cpu-baseline 2>&1 | grep "^{" >> gpurun_out/minb_ab.log
  done
done
