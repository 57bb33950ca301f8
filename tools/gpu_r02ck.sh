mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02ck_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02ck_t.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02ck_smoke.log 2>&1
