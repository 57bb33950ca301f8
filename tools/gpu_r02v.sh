mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "decode or stack or variant or model or lowrank" > gpurun_out/r02v_t.log 2>&1; echo rc=$? >> gpurun_out/r02v_t.log
for i in 1 2; do
DL_LIBRARY=ab DL_XACT=1 timeout 600 python tools/tp_emulate.py --layers 80 --ps 1 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | sed 's/^/xact /' >> gpurun_out/r02v_ab.log
DL_LIBRARY=ab DL_XACT=0 timeout 600 python tools/tp_emulate.py --layers 80 --ps 1 --layouts rp --steps 10 2>&1 | grep -o '"rank_ms_per_step": [0-9.]*' | sed 's/^/silu /' >> gpurun_out/r02v_ab.log
done
