mkdir -p gpurun_out/r2s3_sanitize
for tool in memcheck racecheck synccheck; do for c in s3 fc7; do
timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_probe.py $c > gpurun_out/r2s3_sanitize/r2s3_sanitize_${tool}_${c}.log 2>&1; echo "$tool $c rc=$?"; tail -2 gpurun_out/r2s3_sanitize/r2s3_sanitize_${tool}_${c}.log
done; done
