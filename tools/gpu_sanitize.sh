mkdir -p gpurun_out
tool=${1:-memcheck}
timeout 300 python tools/sanitize_small.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
echo "sanitizer $tool rc=$?"; tail -6 gpurun_out/sanitize_$tool.log
