mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02cj_build.log 2>&1
export DL_LIBRARY=ab
for i in 1 2 3; do for E in "DL_X=0" "DL_DPSK_FRAC=0.9" "DL_DPSK_FRAC=0.5"; do
  echo "[$E] $(env $E timeout 300 python tools/prefill_timeline.py 2>&1 | head -1)"
done; done > gpurun_out/r02cj_ab.log 2>&1
