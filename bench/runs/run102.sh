# re-calibration of the offline table with the round-2 one-pass kernel (first-touch launches), then the
# tail-term measurement on real matrices (bench/calibrate_tail.py) against the new table
set -x
timeout 2400 python bench/calibrate.py > gpurun_out/r02_calibrate_main.log 2>&1; echo main=$?
timeout 1200 python bench/calibrate.py --dram > gpurun_out/r02_calibrate_dram.log 2>&1; echo dram=$?
timeout 1800 python bench/calibrate.py --extend > gpurun_out/r02_calibrate_extend2.log 2>&1; echo extend=$?
python - <<'PY'
import json
p='paper_1103_2405_b200/data/perf_table_b200.json'
t=json.load(open(p)); t['tail_frac']=1.2; json.dump(t, open(p,'w'), indent=0)
json.dump(t, open('gpurun_out/perf_table_b200.json','w'), indent=0)
print('entries', len(t['entries']), 'launch_us', t['launch_us'], 'max_act_warp', t['max_act_warp'])
PY
rm -f gpurun_out/tail2.jsonl
timeout 1800 python bench/calibrate_tail.py --out gpurun_out/tail2.jsonl > gpurun_out/tail2.log 2>&1; echo tail=$?
tail -2 gpurun_out/r02_calibrate_main.log gpurun_out/r02_calibrate_extend2.log
