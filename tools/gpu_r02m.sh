mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill" > gpurun_out/r02m_t.log 2>&1; echo rc=$? >> gpurun_out/r02m_t.log
for c in 1 2; do echo "== C=$c"; DL_LIBRARY=ab DL_FA_CLUSTER=$c timeout 300 python tools/fa_trace.py 2>&1 | tail -8; DL_LIBRARY=ab DL_FA_CLUSTER=$c timeout 300 python tools/prefill_timeline.py 2>&1 | grep attn; done > gpurun_out/r02m_fa.log 2>&1
