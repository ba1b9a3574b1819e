#!/bin/bash
# Run on the GPU box (gpurun).  Produces gpurun_out/prof/* for profiles/<round>/.
# Every ncu command profiles a workload that first ran clean without ncu.
set -x
mkdir -p gpurun_out/prof
CMD="python bench.py --config c2 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-profile"
$CMD > gpurun_out/prof/plain.log 2>&1 || exit 1
DEC="python tools/profile_decode.py --new 88"
$DEC > gpurun_out/prof/decode_plain.log 2>&1 || exit 1
# in-graph timeline of the decode step (CUPTI via torch.profiler): critical-path share per kernel
python tools/timeline.py --new 88 > gpurun_out/prof/timeline_decode.txt 2>&1

# per-stage trace of the decode GEMMs (clock64 inside CTA (0,0))
PPOEXP_GEMM_TRACE=gpurun_out/prof/gemm_trace.bin python tools/profile_decode.py --new 24 > /dev/null 2>&1
python tools/gemm_trace.py gpurun_out/prof/gemm_trace.bin > gpurun_out/prof/gemm_trace.txt 2>&1
# warm-L2 launch list of steady-state decode with DRAM traffic per launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -s 1500 -c 900 --csv --log-file gpurun_out/prof/launches_decode.csv $DEC \
    > gpurun_out/prof/ncu1.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemm_tc|logprob|attn_prefill|layernorm_warp|kv_scatter" -s 420 -c 240 --csv \
    --log-file gpurun_out/prof/launches_scoring.csv $CMD > gpurun_out/prof/ncu2.log 2>&1
# full captures of the top kernels
# gemm_decode launches per decode step: 12 x [QKV, O, up, down] + LM head = 49 (template args do not
# match -k): -s 202 = an O projection (residual + row statistics), -s 201 = a QKV projection (LN fused)
ncu --set full --import-source on --clock-control none -k regex:gemm_decode_kernel -s 202 -c 1 -o gpurun_out/prof/full_gemm_decode $DEC > gpurun_out/prof/ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_decode_kernel -s 201 -c 1 -o gpurun_out/prof/full_gemm_decode_lnin $DEC > gpurun_out/prof/ncu3b.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 100 -c 1 -o gpurun_out/prof/full_attn_decode $DEC > gpurun_out/prof/ncu4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:logprob_gather -s 2 -c 1 -o gpurun_out/prof/full_logprob $CMD > gpurun_out/prof/ncu5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_tc_kernel -s 100 -c 1 -o gpurun_out/prof/full_gemm_tc $CMD > gpurun_out/prof/ncu6.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sampler -s 30 -c 1 -o gpurun_out/prof/full_sampler $DEC > gpurun_out/prof/ncu7.log 2>&1
ls -la gpurun_out/prof
