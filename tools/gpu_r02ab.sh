python tools/gemm_cta_trace.py --tp 8 > gpurun_out/r02ab_g8.log 2>&1
python tools/gemm_cta_trace.py --tp 1 > gpurun_out/r02ab_g1.log 2>&1
