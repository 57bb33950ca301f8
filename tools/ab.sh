#!/bin/bash
# A/B decode-step timing on one box: tools/ab.sh "ENV_A" "ENV_B" [rounds] [extra bench args]
# e.g. tools/ab.sh "" "DL_NO_FUSE_RESNORM=1" 3
A="$1"; B="$2"; R=${3:-3}; shift 3; EXTRA="$@"
for i in $(seq $R); do
  for v in A B; do
    if [ $v = A ]; then E="$A"; else E="$B"; fi
    ms=$(env $E python bench.py --no-cpu-baseline --prefill-tokens 0 --steps 30 $EXTRA 2>/dev/null | tail -1 | \
         python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), round(d['roofline']['frac'],4))")
    echo "$v [$E] $ms"
  done
done
