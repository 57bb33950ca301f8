mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 900 python bench.py > gpurun_out/r02t_bench.log 2>&1
timeout 900 python bench.py --kv lowrank --no-cpu-baseline --prefill-tokens 0 --steps 10 > gpurun_out/r02t_bench_kvlr.log 2>&1
timeout 900 python tools/tp_emulate.py --layers 80 --ps 1,2,4,8 --layouts rp,deinfer --steps 10 > gpurun_out/r02t_tp.log 2>&1
timeout 600 python tools/configs.py > gpurun_out/r02t_configs.log 2>&1
