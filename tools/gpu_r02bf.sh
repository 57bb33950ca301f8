mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bf_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "prefill" > gpurun_out/r02bf_t.log 2>&1; echo rc=$? >> gpurun_out/r02bf_t.log
timeout 300 python tools/prefill_timeline.py > gpurun_out/r02bf_tl.log 2>&1
DL_LIBRARY=ab DL_GLU_FUSE=0 timeout 300 python tools/prefill_timeline.py > gpurun_out/r02bf_tl_off.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02bf_bench.json 2> gpurun_out/r02bf_bench.err
