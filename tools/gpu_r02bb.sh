mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bb_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" > gpurun_out/r02bb_t.log 2>&1; echo rc=$? >> gpurun_out/r02bb_t.log
for rep in 1 2; do
  echo "tc2 $(timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn | awk '{print $NF, $(NF-2)}' | tr '\n' ' ')" >> gpurun_out/r02bb_ab.log
  echo "v1 $(DL_LIBRARY=ab DL_FA_V1=1 timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn | awk '{print $NF, $(NF-2)}' | tr '\n' ' ')" >> gpurun_out/r02bb_ab.log
  for f in 1 2; do
  echo "tc2 fmae=$f $(DL_LIBRARY=ab DL_FA_FMA_EXP=$f timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn | awk '{print $NF, $(NF-2)}' | tr '\n' ' ')" >> gpurun_out/r02bb_ab.log
  done
done
timeout 300 python tools/prefill_timeline.py > gpurun_out/r02bb_tl.log 2>&1
