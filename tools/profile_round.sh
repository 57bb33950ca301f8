#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box via gpurun).  Usage: tools/profile_round.sh <tag>
tag=${1:-r01}
out=gpurun_out
mkdir -p $out
# 1. launch list of the bench command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  -k regex:"tc_gemm|tc_tail|rmsnorm|ew4|silu|rope|attn|embedding|latent|unpermute|gemv|chain|residual|argmax|f32_to" \
  --log-file $out/${tag}_launches_raw.csv python bench.py --steps 2 --warmup 1 --prefill-steps 1 \
  --no-cpu-baseline > $out/${tag}_ncu_bench.log 2>&1
# 2. full sections of the top kernels (one launch each, 2-layer eager steps)
full="--set full --clock-control none --import-source on"
timeout 600 ncu $full -k regex:tc_gemm_kernel -s 13 -c 1 -o $out/${tag}_dec_gu2 -f \
  python tools/step_profile.py --layers 2 --no-prefill > /dev/null 2>&1
timeout 600 ncu $full -k regex:attn_decode -s 1 -c 1 -o $out/${tag}_attn_decode -f \
  python tools/step_profile.py --layers 2 --no-prefill > /dev/null 2>&1
timeout 600 ncu $full -k regex:tc_gemm_pair -s 13 -c 1 -o $out/${tag}_pre_gu2 -f \
  python tools/step_profile.py --layers 2 --no-decode > /dev/null 2>&1
timeout 600 ncu $full -k regex:attn_prefill -s 1 -c 1 -o $out/${tag}_attn_prefill -f \
  python tools/step_profile.py --layers 2 --no-decode > /dev/null 2>&1
ls -la $out
