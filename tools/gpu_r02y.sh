mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 900 python bench.py > gpurun_out/r02y_bench.log 2>&1
