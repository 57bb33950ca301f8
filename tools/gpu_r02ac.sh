python tools/decode_timeline.py --tp 8 --layers 4 > gpurun_out/r02ac_tl8.log 2>&1
