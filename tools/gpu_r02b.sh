set -x
mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 300 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/r02b_chain.log 2>&1; echo rc=$? >> gpurun_out/r02b_chain.log
if grep -q "rc=0" gpurun_out/r02b_chain.log; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gputest.log 2>&1; echo rc=$? >> gpurun_out/r02b_gputest.log
  timeout 300 python bench.py --steps 10 --no-cpu-baseline --prefill-steps 1 > gpurun_out/r02b_bench_chain.log 2>&1
  DL_LIBRARY=ab DL_CHAIN=0 timeout 300 python bench.py --steps 10 --no-cpu-baseline --prefill-steps 1 > gpurun_out/r02b_bench_nochain.log 2>&1
  timeout 300 python bench.py --steps 10 --no-cpu-baseline --prefill-steps 1 > gpurun_out/r02b_bench_chain2.log 2>&1
  timeout 600 python tools/tp_emulate.py --layers 80 --ps 8 --layouts rp --steps 10 > gpurun_out/r02b_tp8.log 2>&1
  DL_LIBRARY=ab DL_CHAIN=0 timeout 600 python tools/tp_emulate.py --layers 80 --ps 8 --layouts rp --steps 10 > gpurun_out/r02b_tp8_nochain.log 2>&1
fi
