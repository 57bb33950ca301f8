mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill and not variants" > gpurun_out/r02m_t.log 2>&1; echo rc=$? >> gpurun_out/r02m_t.log
timeout 300 python tools/fa_trace.py > gpurun_out/r02m_fa.log 2>&1
timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn >> gpurun_out/r02m_fa.log
