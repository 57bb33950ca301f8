mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
full="--set full --clock-control none --import-source on"
timeout 900 ncu $full -k regex:tc_gemm_kernel -s 8 -c 8 -o gpurun_out/r02f_dec_layer -f \
  python tools/step_profile.py --layers 2 --no-prefill > gpurun_out/r02f_ncu.log 2>&1
timeout 600 ncu $full -k regex:attn_decode -s 1 -c 1 -o gpurun_out/r02f_attn_decode -f \
  python tools/step_profile.py --layers 2 --no-prefill >> gpurun_out/r02f_ncu.log 2>&1
ls -la gpurun_out
