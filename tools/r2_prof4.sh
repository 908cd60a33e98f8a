python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu4.log 2>&1
python tools/producers_probe.py > gpurun_out/r2_prod3.json 2>&1
python tools/spmm_probe.py > gpurun_out/r2_spmm4.jsonl 2>&1
for cfg in cfg0 fc7; do
  for tool in memcheck racecheck synccheck; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py $cfg > gpurun_out/r2_sanitize_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$?" >> gpurun_out/r2_sanitize_summary.txt
  done
done
timeout 300 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:spmv_kernel -s 5 -c 2 --csv --log-file gpurun_out/r2_spmv_opld.csv python bench.py --steps 10 --warmup 3 --no-extras > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:spmv_kernel -s 3 -c 1 -o gpurun_out/r2_k4_16384_n8 python tools/spmm_probe.py 16384sq > /dev/null 2>&1
