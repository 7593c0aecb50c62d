#!/bin/bash
# Round-1 measurement refresh on one B200 (run under gpurun): GPU tests, the
# bench lines of both arms, every config, the launch list of the cfg2 step
# and one `ncu --set full` capture of its three main kernels.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r_tests.log 2>&1; tail -2 gpurun_out/r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; tail -c 600 gpurun_out/r_bench.json
timeout 600 python bench.py --impl reference > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err; tail -c 300 gpurun_out/r_bench_ref.json
timeout 600 python bench.py --dist --no-cpu > gpurun_out/r_bench_dist.json 2> gpurun_out/r_bench_dist.err; tail -c 300 gpurun_out/r_bench_dist.json
timeout 900 python tools/bench_configs.py > gpurun_out/r_configs.json 2> gpurun_out/r_configs.err; tail -c 300 gpurun_out/r_configs.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-kv --no-clock-window \
  > gpurun_out/r_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_page_partition_tma|k_page_count|k_emit" -s 3 -c 3 \
  -o gpurun_out/r_full python tools/profile_one.py > gpurun_out/r_ncu_full.log 2>&1; echo "ncu full rc=$?"
