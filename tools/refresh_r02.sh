#!/bin/bash
# Round-2 measurement refresh on one B200 (run under gpurun): GPU tests, smoke,
# the bench line of both arms, the dist path at one rank, the launch list of
# the cfg2 step and one `ncu --set full` capture of its three main kernels.
# Output under gpurun_out/r2/$TAG.
set -u
TAG=${1:-refresh}
O=gpurun_out/r2/$TAG
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/tests.log 2>&1; tail -2 $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 200 $O/bench_ref.json
timeout 900 python bench.py --dist --no-cpu > $O/bench_dist.json 2> $O/bench_dist.err; tail -c 200 $O/bench_dist.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs --no-clock-window > $O/plain_list.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-configs --no-clock-window \
  > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 300 python tools/profile_one.py > $O/plain_full.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_page_partition|k_page_count|k_emit" -s 3 -c 3 \
  -o $O/full python tools/profile_one.py > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
# key/value: launch list and one full capture of the scatter
timeout 600 python tools/profile_one.py --no-cfg2 --kv > $O/plain_kv.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_kv.csv python tools/profile_one.py --no-cfg2 --kv > $O/ncu_kv_launch.log 2>&1; echo "kv launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_kv_chunk_scatter" -s 3 -c 1 \
  -o $O/full_kv python tools/profile_one.py --no-cfg2 --kv > $O/ncu_full_kv.log 2>&1; echo "ncu full kv rc=$?"
