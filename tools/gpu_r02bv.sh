mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bv_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "prefill" > gpurun_out/r02bv_t.log 2>&1; echo rc=$? >> gpurun_out/r02bv_t.log
export DL_LIBRARY=ab
for E in "DL_X=0" "DL_TAIL_KERNEL=1"; do
  echo "[$E] $(env $E timeout 300 python tools/prefill_timeline.py 2>&1 | awk '{print $1, $(NF-2)}' | head -16 | tr '\n' ' ')"
done > gpurun_out/r02bv_ab.log 2>&1
