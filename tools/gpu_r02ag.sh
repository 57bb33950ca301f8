mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ag_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -k "decode" > gpurun_out/r02ag_t.log 2>&1; echo rc=$? >> gpurun_out/r02ag_t.log
python tools/attn_trace.py --tp 8 > gpurun_out/r02ag_attn8.log 2>&1
python tools/attn_trace.py --tp 1 > gpurun_out/r02ag_attn1.log 2>&1
timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 10 2>&1 | grep -o '"P": [0-9]*\|"rank_ms_per_step": [0-9.]*' | paste - - > gpurun_out/r02ag_tp.log
