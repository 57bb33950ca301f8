mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02cd_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "prefill and not variants" > gpurun_out/r02cd_t.log 2>&1; echo rc=$? >> gpurun_out/r02cd_t.log
for i in 1 2; do timeout 300 python tools/prefill_timeline.py 2>&1 | grep -E "step|res\+norm" | head -4 | tr '\n' ' '; echo; done > gpurun_out/r02cd_tl.log 2>&1
