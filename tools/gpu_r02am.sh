mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02am_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_chain.py tests/test_gpu_tp_path.py -x -q 2>&1 | tail -2 > gpurun_out/r02am_t.log
export DL_LIBRARY=ab
run() { echo "[$1] $(env $1 timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,2,4,8 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | paste - - - -)"; }
for i in 1 2; do
  for E in "DL_SK_SMALL=24" "DL_SK_SMALL=0" "DL_SK_SMALL=36" "DL_SK_STATIC_S=0.85" "DL_SK_STATIC_S=0.75" "DL_SK_CHUNK_S=3"; do run "$E"; done
done > gpurun_out/r02am_ab.log 2>&1
