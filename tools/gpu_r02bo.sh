# round 2b results + profiles (one GPU): bench line, TP emulation sweep, configs, ncu
mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bo_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r02bo_bench.json 2> gpurun_out/r02bo_bench.err
timeout 900 python tools/tp_emulate.py --layers 80 --ps 1,2,4,8 --layouts rp,deinfer --steps 10 > gpurun_out/r02bo_tp.jsonl 2> gpurun_out/r02bo_tp.err
timeout 900 python tools/tp_emulate.py --model 8b --layers 0 --ps 1,2,4,8 --layouts rp --steps 10 > gpurun_out/r02bo_tp8b.jsonl 2> gpurun_out/r02bo_tp8b.err
timeout 600 python tools/configs.py > gpurun_out/r02bo_configs.jsonl 2> gpurun_out/r02bo_configs.err
timeout 900 python bench.py --kv lowrank --no-cpu-baseline > gpurun_out/r02bo_kvlr.json 2> gpurun_out/r02bo_kvlr.err
timeout 300 python tools/prefill_timeline.py > gpurun_out/r02bo_prefill_tl.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02bo_decode_tl.log 2>&1
bash tools/profile_round.sh r02b > gpurun_out/r02bo_prof.log 2>&1
