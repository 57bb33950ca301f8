mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill or decode_small or variant" > gpurun_out/r02x_t.log 2>&1; echo rc=$? >> gpurun_out/r02x_t.log
timeout 300 python tools/prefill_timeline.py > gpurun_out/r02x_ptl.log 2>&1
