mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
S="compute-sanitizer --print-limit 10"
timeout 900 $S --tool synccheck python -m pytest -x -q tests/test_gpu_parity.py -k "block_prefill_small or block_decode_small" > gpurun_out/r02s_sync.log 2>&1; echo rc=$? >> gpurun_out/r02s_sync.log
timeout 600 python -m pytest -x -q tests/test_gpu_parity.py -k "prefill" > gpurun_out/r02s_t.log 2>&1; echo rc=$? >> gpurun_out/r02s_t.log
timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn > gpurun_out/r02s_ptl.log
