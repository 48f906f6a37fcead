mkdir -p gpurun_out
timeout 600 python -m pytest tests/ -q -m gpu -x -k "offsets or ragged" > gpurun_out/pytest_off.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_off.log; tail -n 2 gpurun_out/pytest_off.log
timeout 120 python tools/offsets_rate.py > gpurun_out/offsets.jsonl 2>&1; cat gpurun_out/offsets.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"offsets" --csv python tools/offsets_rate.py 2>/dev/null | grep -E "offsets_" | head -4 | awk -F'","' '{print $5, $NF}'
