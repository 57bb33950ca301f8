mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ai_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_tp_path.py tests/test_gpu_peer.py -x -q 2>&1 | tail -3 > gpurun_out/r02ai_t.log
DL_ROPE_FUSE_TP=0 timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q -k decode 2>&1 | tail -1 >> gpurun_out/r02ai_t.log
for i in 1 2; do for M in 0 1; do
  echo "F=$M $(DL_ROPE_FUSE_TP=$M timeout 600 python tools/tp_emulate.py --layers 80 --ps 2,4,8 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | paste - - -)"
done; done > gpurun_out/r02ai_tp.log
python tools/decode_timeline.py --tp 8 --layers 2 > gpurun_out/r02ai_tl8.log 2>&1
