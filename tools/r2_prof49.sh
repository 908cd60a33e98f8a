mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu49.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2_gpu49.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke49.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2_smoke49.log
