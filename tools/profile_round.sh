#!/bin/bash
# Run on the GPU box (gpurun).  Produces gpurun_out/prof/* for profiles/<round>/.
set -x
mkdir -p gpurun_out/prof
CMD="python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-profile"
$CMD > gpurun_out/prof/plain.log 2>&1 || exit 1
# launch list over part of the timed step's decode (skip warm-up + prefill) and its scoring kernels
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -s 30000 -c 3000 --csv \
    --log-file gpurun_out/prof/launches_decode.csv $CMD > gpurun_out/prof/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemm_tc|logprob|attn_prefill|layernorm_warp|kv_scatter" -s 420 -c 240 --csv \
    --log-file gpurun_out/prof/launches_scoring.csv $CMD > gpurun_out/prof/ncu2.log 2>&1
# full captures of the top kernels (decode GEMM, decode attention, K9 log-prob, scoring GEMM, sampler)
ncu --set full --import-source on --clock-control none -k regex:gemm_decode_kernel -s 2000 -c 1 -o gpurun_out/prof/full_gemm_decode $CMD > gpurun_out/prof/ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 1000 -c 1 -o gpurun_out/prof/full_attn_decode $CMD > gpurun_out/prof/ncu4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:logprob_gather -s 2 -c 1 -o gpurun_out/prof/full_logprob $CMD > gpurun_out/prof/ncu5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 100 -c 1 -o gpurun_out/prof/full_gemm_tc $CMD > gpurun_out/prof/ncu6.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sampler -s 300 -c 1 -o gpurun_out/prof/full_sampler $CMD > gpurun_out/prof/ncu7.log 2>&1
ls -la gpurun_out/prof
