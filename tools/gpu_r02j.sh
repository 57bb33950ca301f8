mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
run() { echo "== $*"; env DL_LIBRARY=ab "$@" timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 10 2>&1 | grep -o '"P": [0-9]*\|"rank_ms_per_step": [0-9.]*' | paste - - ; }
{
for i in 1 2; do
run DL_ATTN_ORDER=1
run DL_ATTN_ORDER=0
done
} > gpurun_out/r02j_ab.log 2>&1
