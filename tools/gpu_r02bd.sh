mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bd_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill and not variants" > gpurun_out/r02bd_t.log 2>&1; echo rc=$? >> gpurun_out/r02bd_t.log
for rep in 1 2; do
  echo "tc2 $(timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn | awk '{print $NF, $(NF-2)}' | tr '\n' ' ')" >> gpurun_out/r02bd_ab.log
  echo "v1 $(DL_LIBRARY=ab DL_FA_V1=1 timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn | awk '{print $NF, $(NF-2)}' | tr '\n' ' ')" >> gpurun_out/r02bd_ab.log
done
{ echo "== tc2"; timeout 300 python tools/fa_trace.py; } > gpurun_out/r02bd_fa.log 2>&1
