set -x
mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 600 python tools/tp_emulate.py --layers 80 --ps 8 --layouts rp --steps 10 > gpurun_out/r02d_tp8.log 2>&1
DL_LIBRARY=ab DL_CHAIN=0 timeout 600 python tools/tp_emulate.py --layers 80 --ps 8 --layouts rp --steps 10 > gpurun_out/r02d_tp8_nochain.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 --tp 8 > gpurun_out/r02d_tl8_chain.log 2>&1
DL_LIBRARY=ab DL_CHAIN=0 timeout 300 python tools/decode_timeline.py --layers 4 --tp 8 > gpurun_out/r02d_tl8_nochain.log 2>&1
