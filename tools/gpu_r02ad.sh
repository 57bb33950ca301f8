for i in 1 2 3; do
  for E in "DL_CHAIN=0" "DL_CHAIN=1" "DL_CHAIN=1 DL_CHAIN_PF=0"; do
    echo "[$E] $(env $E python tools/tp_emulate.py --ps 8 --layouts rp 2>/dev/null | tail -1)"
  done
done > gpurun_out/r02ad_ab.log 2>&1
DL_CHAIN=1 python tools/decode_timeline.py --tp 8 --layers 2 > gpurun_out/r02ad_tl8c.log 2>&1
