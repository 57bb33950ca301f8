mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
full="--set full --clock-control none --import-source on"
timeout 600 ncu $full -k regex:attn_decode -s 2 -c 1 -o gpurun_out/r02g_attn_tp8 -f \
  python tools/decode_timeline.py --layers 2 --tp 8 > gpurun_out/r02g_ncu.log 2>&1
