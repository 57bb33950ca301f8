mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02cp_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_tp_path.py tests/test_gpu_fullsize.py -x -q -k "decode or multirank or stack or graph or lowrank" > gpurun_out/r02cp_t.log 2>&1; echo rc=$? >> gpurun_out/r02cp_t.log
export DL_LIBRARY=ab
for i in 1 2 3; do for E in "DL_X=0" "DL_ATTN_ZERO_LATE=0"; do
  echo "[$E] $(env $E timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 20 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | awk '{print $2}' | tr '\n' ' ')"
done; done > gpurun_out/r02cp_ab.log 2>&1
