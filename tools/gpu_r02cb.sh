# final round-2b results: bench line, TP sweep, ncu launch list + top kernels
mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02cb_build.log 2>&1
timeout 900 python bench.py > gpurun_out/r02cb_bench.json 2> gpurun_out/r02cb_bench.err
timeout 900 python tools/tp_emulate.py --layers 80 --ps 1,2,4,8 --layouts rp,deinfer --steps 10 > gpurun_out/r02cb_tp.jsonl 2> gpurun_out/r02cb_tp.err
timeout 300 python tools/attn_trace.py > gpurun_out/r02cb_attn_trace.log 2>&1
timeout 300 python tools/decode_timeline.py --layers 4 > gpurun_out/r02cb_decode_tl.log 2>&1
bash tools/profile_round.sh r02c > gpurun_out/r02cb_prof.log 2>&1
