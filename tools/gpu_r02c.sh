set -x
mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -x -q > gpurun_out/r02c_t.log 2>&1; echo rc=$? >> gpurun_out/r02c_t.log
timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02c_tl_chain.log 2>&1
DL_LIBRARY=ab DL_CHAIN=0 timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02c_tl_nochain.log 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --prefill-steps 1 > gpurun_out/r02c_bench_chain.log 2>&1
DL_LIBRARY=ab DL_CHAIN=0 timeout 300 python bench.py --steps 10 --no-cpu-baseline --prefill-steps 1 > gpurun_out/r02c_bench_nochain.log 2>&1
