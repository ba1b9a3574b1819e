mkdir -p gpurun_out/scale2
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/scale2/s_c2_$n.log 2>&1
  tail -1 gpurun_out/scale2/s_c2_$n.log | head -c 200; echo
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29650 bench.py --gpus 4 --config c3 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/scale2/s_c3_4.log 2>&1
tail -1 gpurun_out/scale2/s_c3_4.log | head -c 200
