#!/bin/bash
# Round-2 profiles (run on the GPU box through gpurun).  Produces gpurun_out/prof2/*
# for profiles/round2/.  Every ncu command profiles a workload that first ran
# clean without ncu; --clock-control none throughout (B200_PROFILING.md).
set -x
O=gpurun_out/prof2
R=/tmp/prof2rep   # full reports stay on the box; their csv pages come back
mkdir -p $O $R
BENCH="python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-profile --no-variant"
$BENCH > $O/bench_plain.log 2>&1 || exit 1
DEC="python tools/profile_decode.py --new 88 --dtype mixed"
$DEC > $O/decode_plain.log 2>&1 || exit 1
SCORE="python tools/profile_decode.py --new 24 --dtype mixed --score 1"
$SCORE > $O/score_plain.log 2>&1 || exit 1
# 1. the contract's launch list of the bench command (per-launch device times, cold, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv $BENCH > $O/ncu0.log 2>&1
# 2. warm-L2 launch list of steady-state mixed decode with DRAM bytes per launch
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none -s 1500 -c 900 --csv --log-file $O/launches_decode.csv $DEC > $O/ncu1.log 2>&1
# 3. scoring-phase kernels with DRAM bytes
SCO="python tools/profile_score.py --reps 2"
$SCO > $O/score_only_plain.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"gemm_pp|attn_prefill|layernorm|lse_combine|embed|logprob" -s 100 -c 100 --csv --log-file $O/launches_scoring.csv $SCO > $O/ncu2.log 2>&1
# 4. full captures of the top kernels
ncu --set full --import-source on --clock-control none -k regex:gemm_decode_kernel -s 202 -c 1 -o $R/full_gemm_decode_a $DEC > $O/ncu3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gemm_decode_kernel -s 201 -c 1 -o $R/full_gemm_decode_b $DEC > $O/ncu4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_decode -s 100 -c 1 -o $R/full_attn_decode $DEC > $O/ncu5.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sampler -s 30 -c 1 -o $R/full_sampler $DEC > $O/ncu6.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"gemm_pp_kernel" -s 60 -c 1 -o $R/full_gemm_pp $SCO > $O/ncu7.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"attn_prefill_split" -s 10 -c 1 -o $R/full_attn_prefill_split $SCORE > $O/ncu8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"layernorm_split" -s 30 -c 1 -o $R/full_ln_split $SCO > $O/ncu9.log 2>&1
# bf16 scoring: tcgen05 flash attention (C2 shape) and the C5-shape launch
BSCORE="python tools/profile_decode.py --new 24 --dtype bf16 --score 1"
$BSCORE > $O/bscore_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"attn_prefill_tc" -s 10 -c 1 -o $R/full_attn_prefill_tc $BSCORE > $O/ncu10.log 2>&1
python tools/profile_attn.py 0 > $O/attn_c5_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"attn_prefill_tc" -s 3 -c 1 -o $R/full_attn_prefill_tc_c5 python tools/profile_attn.py 0 > $O/ncu11.log 2>&1
# export each full report (raw metrics + source pages); bring back reports while under ~40 MB
for r in $R/*.ncu-rep; do
  n=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > $O/${n}_raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $O/${n}_details.csv 2>/dev/null
  ncu -i $r --page source --csv > $O/${n}_source.csv 2>/dev/null
  if [ $(du -sm $O | cut -f1) -lt 40 ]; then cp $r $O/; fi
done
ls -la $O
