mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" > gpurun_out/r02l_t.log 2>&1; echo rc=$? >> gpurun_out/r02l_t.log
timeout 300 python tools/prefill_timeline.py > gpurun_out/r02l_ptl_tc.log 2>&1
full="--set full --clock-control none --import-source on"
timeout 600 ncu $full -k regex:attn_prefill -s 1 -c 1 -o gpurun_out/r02l_attn_prefill -f \
  python tools/step_profile.py --layers 2 --no-decode > gpurun_out/r02l_ncu.log 2>&1
