mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ah_build.log 2>&1
for M in 3 2 1; do DL_ATTN_MERGE=$M timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -k "decode" 2>&1 | tail -1; done > gpurun_out/r02ah_t.log 2>&1
for i in 1 2; do for M in 0 1 2 3; do
  echo "M=$M $(DL_ATTN_MERGE=$M timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | paste - -)"
done; done > gpurun_out/r02ah_tp.log
for M in 0 3; do DL_ATTN_MERGE=$M python tools/attn_trace.py --tp 1 > gpurun_out/r02ah_attn1_$M.log 2>&1; DL_ATTN_MERGE=$M python tools/attn_trace.py --tp 8 > gpurun_out/r02ah_attn8_$M.log 2>&1; done
