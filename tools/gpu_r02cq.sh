mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02cq_build.log 2>&1
export DL_LIBRARY=ab
for i in 1 2 3; do for E in "DL_X=0" "DL_ROPE_FUSE_TP=0"; do
  echo "[$E] $(env $E timeout 600 python tools/tp_emulate.py --layers 80 --ps 2,4,8 --layouts rp --steps 20 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | awk '{print $2}' | tr '\n' ' ')"
done; done > gpurun_out/r02cq_ab.log 2>&1
