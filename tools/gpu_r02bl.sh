mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bl_build.log 2>&1
export DL_LIBRARY=ab
for E in "DL_X=0" "DL_ATTN_TILES_PER_CTA=5" "DL_ATTN_TILES_PER_CTA=6" "DL_ATTN_TILES_PER_CTA=9" "DL_ATTN_TILES_PER_CTA=12"; do
  echo "[$E tp8] $(env $E timeout 300 python tools/attn_trace.py --tp 8 2>&1 | tail -4 | tr '\n' ' ')"
  echo "[$E tp4] $(env $E timeout 300 python tools/attn_trace.py --tp 4 2>&1 | tail -4 | tr '\n' ' ')"
done > gpurun_out/r02bl_ab.log 2>&1
for E in "DL_X=0" "DL_ATTN_TILES_PER_CTA=6" "DL_ATTN_TILES_PER_CTA=9"; do
  echo "[$E] $(env $E timeout 600 python tools/tp_emulate.py --layers 80 --ps 4,8 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | paste - -)"
done >> gpurun_out/r02bl_ab.log 2>&1
