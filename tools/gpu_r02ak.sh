mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ak_build.log 2>&1
export DL_LIBRARY=ab
run() { echo "[$1] $(env $1 timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | paste - -)"; }
for i in 1 2; do
  for E in "DL_ROPE_FUSE_TP=1" "DL_ROPE_FUSE_TP=0" "DL_XACT_TP=1" "DL_CHAIN=1" "DL_SK_STATIC=1.0" "DL_SK_CHUNK=1" "DL_SK_STATIC=0.8 DL_SK_CHUNK=2"; do run "$E"; done
done > gpurun_out/r02ak_ab.log 2>&1
