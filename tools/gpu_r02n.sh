mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02n_gputest.log 2>&1; echo rc=$? >> gpurun_out/r02n_gputest.log
timeout 600 python bench.py > gpurun_out/r02n_bench.log 2>&1
full="--set full --clock-control none --import-source on"
timeout 600 ncu $full -k regex:attn_prefill -s 1 -c 1 -o gpurun_out/r02n_attn_prefill -f \
  python tools/step_profile.py --layers 2 --no-decode > gpurun_out/r02n_ncu.log 2>&1
