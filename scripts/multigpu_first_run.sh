#!/bin/bash
# First run on a multi-GPU box (none was available in rounds 1-2): parity of the NCCL / P2P /
# NVLS sharded steps on real peers, then the bench at every N the box allows, with NCCL's own
# algorithm choice recorded (NVLS vs ring).  Logs in gpurun_out/mg/.  Run from the repo root.
set -u
mkdir -p gpurun_out/mg
NG=$(nvidia-smi -L | wc -l)
echo "GPUs: $NG" | tee gpurun_out/mg/summary.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/mg/build.log 2>&1
port=29611
for N in 2 4 8; do
  [ "$N" -le "$NG" ] || continue
  port=$((port + 10))
  timeout 900 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port \
      -m pytest tests/test_multigpu.py -q -p no:cacheprovider > gpurun_out/mg/test_N$N.log 2>&1
  echo "N=$N tests rc=$? $(tail -1 gpurun_out/mg/test_N$N.log)" | tee -a gpurun_out/mg/summary.txt
  port=$((port + 10))
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,TUNING timeout 1200 python -m torch.distributed.run --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 20 --warmup 5 \
      > gpurun_out/mg/bench_N$N.log 2> gpurun_out/mg/bench_N$N.err
  echo "N=$N bench rc=$?" | tee -a gpurun_out/mg/summary.txt
  grep -m 5 -i "nvls" gpurun_out/mg/bench_N$N.err | tee -a gpurun_out/mg/summary.txt
  grep '^{' gpurun_out/mg/bench_N$N.log | cut -c1-400 | tee -a gpurun_out/mg/summary.txt
done
