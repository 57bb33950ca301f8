mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
run() { echo "== $*"; env DL_LIBRARY=ab "$@" timeout 600 python tools/tp_emulate.py --layers 80 --ps 8 --layouts rp --steps 10 2>&1 | grep -o '"P": [0-9]*\|"rank_ms_per_step": [0-9.]*' | paste - - ; }
{
run DL_X=0
run DL_DECODE_STAGES=4
run DL_DECODE_STAGES=4 DL_DECODE_PER_SM=1
run DL_CHAIN=1
run DL_CHAIN=1 DL_CHAIN_WARP=1
run DL_X=0
} > gpurun_out/r02q_ab.log 2>&1
