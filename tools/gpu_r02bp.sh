# sanitizers on the round-2b paths + config 5 sweep
mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bp_build.log 2>&1
S="compute-sanitizer --print-limit 10"
# GLU pair kernel + RoPE epilogue + copy-only append (prefill, T = 300 / 400 / 2 seq), decode attention no-split + deep ring
timeout 1200 $S --tool memcheck python -m pytest -x -q tests/test_gpu_parity.py -k "block_prefill_small or block_decode_small or cached_prefix" > gpurun_out/r02bp_mem.log 2>&1; echo rc=$? >> gpurun_out/r02bp_mem.log
timeout 1200 $S --tool synccheck python -m pytest -x -q tests/test_gpu_parity.py -k "block_prefill_small or block_decode_small" > gpurun_out/r02bp_sync.log 2>&1; echo rc=$? >> gpurun_out/r02bp_sync.log
timeout 1200 $S --tool racecheck python -m pytest -x -q tests/test_gpu_parity.py -k "block_prefill_small" > gpurun_out/r02bp_race.log 2>&1; echo rc=$? >> gpurun_out/r02bp_race.log
timeout 1200 $S --tool memcheck python -m pytest -x -q tests/test_gpu_multirank.py -k "decode and 4" > gpurun_out/r02bp_mem_mr.log 2>&1; echo rc=$? >> gpurun_out/r02bp_mem_mr.log
timeout 1500 python tools/tp_emulate.py --layers 80 --ps 2,4,8 --layouts rp --ratios 0.1,0.2,0.3,0.4,0.5,0.6 --steps 10 > gpurun_out/r02bp_cfg5.jsonl 2> gpurun_out/r02bp_cfg5.err
