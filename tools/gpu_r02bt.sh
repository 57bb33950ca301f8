mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bt_build.log 2>&1
timeout 900 env DL_LIBRARY=ab DL_SK_GUIDED=1 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chain.py -x -q -k "decode or chain" > gpurun_out/r02bt_t.log 2>&1; echo rc=$? >> gpurun_out/r02bt_t.log
export DL_LIBRARY=ab
for i in 1 2; do for E in "DL_X=0" "DL_SK_GUIDED=1" "DL_SK_GUIDED=2" "DL_SK_GUIDED=1 DL_SK_CHUNK=16" "DL_SK_GUIDED=1 DL_SK_STATIC=0.8 DL_SK_CHUNK=16"; do
  echo "[$E] $(env $E timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 20 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | awk '{print $2}' | tr '\n' ' ')"
done; done > gpurun_out/r02bt_ab.log 2>&1
