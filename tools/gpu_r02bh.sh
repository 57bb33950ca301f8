mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bh_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02bh_t.log
timeout 900 python bench.py > gpurun_out/r02bh_bench.json 2> gpurun_out/r02bh_bench.err
