mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "wavefront or graph" > gpurun_out/r02r_t.log 2>&1; echo rc=$? >> gpurun_out/r02r_t.log
for c in 1 2 4 1 2; do timeout 600 python bench.py --steps 5 --no-cpu-baseline --prefill-steps 3 --prefill-chunks $c > gpurun_out/r02r_b$c.log 2>&1; python -c "
import json
l=[x for x in open('gpurun_out/r02r_b$c.log') if x.startswith('{')]
d=json.loads(l[-1]); p=d['prefill']; print('chunks', p['chunks'], 'prefill ms', round(p['ms_per_step'],2), 'decode ms', round(d['ms_per_step'],2), 'in-graph', d['roofline'].get('gemm_class_in_graph'))" >> gpurun_out/r02r_sum.log 2>&1; done
