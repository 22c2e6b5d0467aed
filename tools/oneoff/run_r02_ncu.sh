# r02: full ncu captures of the decode launch; summaries, raw metrics and (C5) the SASS source page
# are written to gpurun_out/ and the .ncu-rep files removed (gpurun brings back <= 64 MiB)
mkdir -p gpurun_out
./tools/microbench_ffma2 > gpurun_out/p_ffma2.txt 2>&1
K="regex:band_kernel|xband"
cap() {  # tag, bench args...
  tag=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -o /tmp/ncu_$tag -f python bench.py "$@" --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/ncu_$tag.log 2>&1
  python tools/ncu_summary.py full /tmp/ncu_$tag.ncu-rep > gpurun_out/ncu_$tag.txt 2>&1
  ncu -i /tmp/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_raw.csv 2>&1
  if [ "$SRC" = 1 ]; then ncu -i /tmp/ncu_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${tag}_sass.csv 2>&1; fi
  rm -f /tmp/ncu_$tag.ncu-rep
}
SRC=1 cap c5 --config C5 --frames 16384
SRC=1 cap c2 --config C2 --ebn0 1.0
cap c3r12 --config C3-R1/2
SRC=1 cap c4 --frames 32768
cap t1r14 --config T1-R1/4 --frames 1000
