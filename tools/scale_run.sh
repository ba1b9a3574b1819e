#!/bin/bash
# Builder-side scaling runs on one box (gpurun --gpus N): c2 weak, c3 strong.
# Output: gpurun_out/scale/s_<config>_<N>.log (the JSON line is the last line).
N=${1:-4}
O=gpurun_out/scale
mkdir -p $O
run() {  # config, gpus, extra args
  if [ "$2" = "1" ]; then
    timeout 1200 python bench.py --config $1 ${@:3} > $O/s_$1_$2.log 2>&1
  else
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $2 --master-addr 127.0.0.1 \
      --master-port $((29500 + $2)) bench.py --gpus $2 --config $1 ${@:3} > $O/s_$1_$2.log 2>&1
  fi
  tail -1 $O/s_$1_$2.log | head -c 160; echo
}
for n in $(seq 2 $N); do
  if [ $n = 2 ] || [ $n = 4 ] || [ $n = 8 ]; then
    run c2 $n --steps 10 --warmup 3 --no-cpu-baseline
    run c3 $n --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline
  fi
done
run c3 1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline
run c4 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline
