python -m pytest tests/test_gpu_parity.py tests/test_gpu_patterns.py -m gpu -q -x -k "prune or pack or rank or random or small or special or full" > gpurun_out/r2_gpuprod.log 2>&1
python tools/producers_probe.py > gpurun_out/r2_prod1.json 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prune_thread -s 1 -c 1 -o gpurun_out/r2_prune2 python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:block_rank -c 1 -o gpurun_out/r2_brank2 python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pack_row -c 1 -o gpurun_out/r2_pack2 python tools/producers_probe.py 16384 65536 3 > /dev/null 2>&1
