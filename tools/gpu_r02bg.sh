mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bg_build.log 2>&1
export DL_LIBRARY=ab
run() { echo "[$1] $(env $1 timeout 300 python tools/prefill_timeline.py 2>&1 | grep -E 'step|silu|gemm' | sed -n '1p;9,12p' | awk '{print $NF=="us"?$0:$(NF-2)}' | tr '\n' ' ')"; }
for i in 1 2; do
  for E in "DL_X=0" "DL_GLU_FUSE=0" "DL_GLU_ACT_POL=1" "DL_GLU_WPOL=1" "DL_GLU_WPOL=1 DL_GLU_ACT_POL=1" "DL_GLU_WPOL=0 DL_GLU_ACT_POL=1"; do run "$E"; done
done > gpurun_out/r02bg_ab.log 2>&1
