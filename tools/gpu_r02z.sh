mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
for rep in 1 2; do for f in 0 1 2; do
  echo "fmae=$f $(DL_LIBRARY=ab DL_FA_FMA_EXP=$f timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn | awk '{print $NF, $(NF-2)}' | tr '\n' ' ')" >> gpurun_out/r02z_fma.log
done; done
DL_LIBRARY=ab DL_FA_FMA_EXP=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "block_prefill_small or cached_prefix" > gpurun_out/r02z_t.log 2>&1; echo rc=$? >> gpurun_out/r02z_t.log
