mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bk_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r02bk_t.log
