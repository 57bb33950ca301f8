mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" > gpurun_out/r02k_t.log 2>&1; echo rc=$? >> gpurun_out/r02k_t.log
