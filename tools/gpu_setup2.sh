# K4 + seg layout build: full GPU suite, setup launch list (C4), C4 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/setup4_c4.csv python tools/setup_breakdown.py c4 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_list.py gpurun_out/setup4_c4.csv 200 | grep -v "k_fy\|k_gg\|scan_apply\|k_random_rows"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/setup4_c3.csv python tools/setup_breakdown.py c3 > /dev/null 2>&1; echo ncu rc=$?
python tools/ncu_list.py gpurun_out/setup4_c3.csv 200 | grep -v "k_fy\|k_gg\|scan_apply\|rmat"
timeout 900 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1]); print({k:d.get(k) for k in ['value','ms_per_step','permute_ms','permute_warm_ms','seg_build_ms','hist_ms']}); print(d.get('setup'))"
