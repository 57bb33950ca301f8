mkdir -p gpurun_out
python -m paper_2604_17709_b200.build > /dev/null
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02w_gputest.log 2>&1; echo rc=$? >> gpurun_out/r02w_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02w_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02w_smoke.log
