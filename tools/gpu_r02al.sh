mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02al_build.log 2>&1
export DL_LIBRARY=ab
run() { echo "[$1] $(env $1 timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,4,8 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | paste - - -)"; }
for i in 1 2; do
  for E in "DL_SK_SMALL=0" "DL_SK_SMALL=24" "DL_SK_STATIC_S=0.7" "DL_SK_STATIC_S=0.8 DL_SK_CHUNK_S=1" "DL_SK_STATIC_S=0.6 DL_SK_CHUNK_S=2" "DL_SK_STATIC_S=0.8 DL_SK_CHUNK_S=4" "DL_SK_SMALL=12" "DL_SK_SMALL=48"; do run "$E"; done
done > gpurun_out/r02al_ab.log 2>&1
