mkdir -p gpurun_out
K="regex:band_kernel|xband"
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -c 1 -o /tmp/n4 -f python bench.py --frames 32768 --steps 1 --warmup 0 --eager --no-cpu-baseline --no-e2e > gpurun_out/n4.log 2>&1
python tools/ncu_summary.py full /tmp/n4.ncu-rep > gpurun_out/n4.txt 2>&1
ncu -i /tmp/n4.ncu-rep --page source --csv --print-source sass > gpurun_out/n4_sass.csv 2>&1
rm -f /tmp/n4.ncu-rep
