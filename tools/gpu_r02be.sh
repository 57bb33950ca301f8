mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02be_build.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 --tp 8 > gpurun_out/r02be_tl8.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02be_tl1.log 2>&1
timeout 300 python tools/gemm_cta_trace.py --tp 8 > gpurun_out/r02be_cta8.log 2>&1
