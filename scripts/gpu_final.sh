#!/bin/bash
# Round-end evidence on one B200: parity tests, smoke, bench line (+ torchrun
# N=1 and the reference arm), launch list of the bench command, per-config report.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err
echo "torchrun exit $?" >> gpurun_out/bench_torchrun.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref exit $?" >> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
python profiles/summarize_launches.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench.txt
timeout 900 python scripts/config_report.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -n 1 gpurun_out/bench.err gpurun_out/bench_torchrun.err gpurun_out/bench_ref.err
cut -c1-300 gpurun_out/bench.json gpurun_out/bench_torchrun.json gpurun_out/bench_ref.json; cat gpurun_out/launches_bench.txt; cut -c1-250 gpurun_out/configs.jsonl
