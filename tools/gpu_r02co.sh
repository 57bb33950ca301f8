mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02co_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/r02co_t.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02co_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02co_bench.json 2> gpurun_out/r02co_bench.err
timeout 900 python tools/tp_emulate.py --layers 80 --ps 1,2,4,8 --layouts rp,deinfer --steps 10 > gpurun_out/r02co_tp.jsonl 2> gpurun_out/r02co_tp.err
