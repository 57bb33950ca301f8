mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bz_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_fullsize.py -x -q -k "decode or multirank or stack" > gpurun_out/r02bz_t.log 2>&1; echo rc=$? >> gpurun_out/r02bz_t.log
timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02bz_tl1.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 --tp 8 > gpurun_out/r02bz_tl8.log 2>&1
timeout 600 python tools/tp_emulate.py --layers 80 --ps 1,8 --layouts rp --steps 20 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' > gpurun_out/r02bz_tp.log
