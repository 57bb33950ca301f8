mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ci_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "prefill and not variants" > gpurun_out/r02ci_t.log 2>&1; echo rc=$? >> gpurun_out/r02ci_t.log
export DL_LIBRARY=ab
for i in 1 2 3; do for E in "DL_X=0" "DL_RMS_2P=0"; do
  echo "[$E] $(env $E timeout 300 python tools/prefill_timeline.py 2>&1 | grep -E 'step|res\+norm' | head -4 | awk '{print $1, $2, $3, $(NF-2)}' | tr '\n' ' ')"
done; done > gpurun_out/r02ci_ab.log 2>&1
