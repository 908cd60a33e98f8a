set -x
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "random_shapes or small or unit or sixteen or pass_widths" > gpurun_out/r2_gpurand.log 2>&1
python tools/producers_probe.py > gpurun_out/r2_prod0.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prune_thread -s 1 -c 1 -o gpurun_out/r2_prune python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:block_rank -c 1 -o gpurun_out/r2_brank python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pack_kernel -c 1 -o gpurun_out/r2_pack python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
ls -la gpurun_out/
