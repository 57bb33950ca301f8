mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ch_build.log 2>&1
timeout 300 python tools/prefill_timeline.py --layers 2 > gpurun_out/r02ch_prefill_tl.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02ch_decode_tl.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 --tp 8 > gpurun_out/r02ch_decode_tl8.log 2>&1
