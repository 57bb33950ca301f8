mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_gputest.log 2>&1; echo rc=$? >> gpurun_out/r02i_gputest.log
timeout 600 python bench.py > gpurun_out/r02i_bench.log 2>&1
