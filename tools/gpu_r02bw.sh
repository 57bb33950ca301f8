mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bw_build.log 2>&1
export DL_LIBRARY=ab
for i in 1 2; do for E in "DL_X=0" "DL_DECODE_STAGES=4" "DL_DECODE_STAGES=4 DL_DECODE_PER_SM=1" "DL_SK_STATIC_S=1.0" "DL_CHAIN=1" "DL_SK_CHUNK_S=2"; do
  echo "[$E] $(env $E timeout 600 python tools/tp_emulate.py --layers 80 --ps 4,8 --layouts rp --steps 20 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | awk '{print $2}' | tr '\n' ' ')"
done; done > gpurun_out/r02bw_ab.log 2>&1
