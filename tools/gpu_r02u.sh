mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 600 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/r02u_peer.log 2>&1; echo rc=$? >> gpurun_out/r02u_peer.log
