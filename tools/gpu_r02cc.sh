mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > gpurun_out/r02cc_build.log 2>&1
export DL_LIBRARY=ab
for i in 1 2; do for E in "DL_GLU_WPOL=0" "DL_GLU_WPOL=2"; do
  env $E timeout 900 python bench.py --steps 5 --warmup 3 --prefill-steps 6 --no-cpu-baseline > gpurun_out/r02cc_b.json 2>/dev/null
  echo "[$E] $(python -c "
import json; d=json.loads(open('gpurun_out/r02cc_b.json').read().strip().splitlines()[-1]); p=d['prefill']; print(p['ms_per_step'], p['clocks']['sm_mhz'], p['clocks']['power_w_max'])")"
done; done > gpurun_out/r02cc_ab.log 2>&1
