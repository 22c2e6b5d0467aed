# full GPU test suite + smoke + issue profile of every workload + default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/full_tests.log 2>&1; echo EXIT $? >> gpurun_out/full_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo EXIT $? >> gpurun_out/full_smoke.log
timeout 2400 python tools/issue_profile.py gpurun_out/issue_full.json > gpurun_out/full_issue.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/full_bench.log 2>&1
