#!/bin/bash
# Prefill weight L2-policy A/B (DL_PAIR_WPOL 0 = evict_first, 1 = normal, 2 = last): in-graph
# 2-layer prefill step time and DRAM bytes of the gate|up stage-2 launch (run on the GPU box).
for v in 0 1 2; do echo "WPOL=$v"; DL_PAIR_WPOL=$v python tools/prefill_timeline.py --layers 2 2>&1 | head -1; done
for v in 0 1 2; do DL_PAIR_WPOL=$v timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:tc_gemm_pair -s 5 -c 1 --csv python tools/step_profile.py --layers 1 --no-decode 2>/dev/null | tail -2 | cut -c1-250; done
