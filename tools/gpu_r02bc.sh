mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02bc_build.log 2>&1
{ echo "== tc2"; timeout 300 python tools/fa_trace.py; echo "== v1"; DL_LIBRARY=ab DL_FA_V1=1 timeout 300 python tools/fa_trace.py; } > gpurun_out/r02bc_fa.log 2>&1
