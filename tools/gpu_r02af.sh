for i in 1 2; do
  for E in "DL_SK_STATIC=0.9" "DL_SK_STATIC=1.0" ; do
    echo "[$E] $(env $E python tools/tp_emulate.py --ps 1,8 --layouts rp --steps 10 2>/dev/null | python -c "
import sys,json
print(' '.join(f\"P{d['P']}={d['rank_ms_per_step']}\" for d in map(json.loads, [l for l in sys.stdin if l.startswith('{')])))")"
  done
done > gpurun_out/r02af_ab.log 2>&1
DL_SK_STATIC=1.0 python tools/gemm_cta_trace.py --tp 8 > gpurun_out/r02af_g8.log 2>&1
