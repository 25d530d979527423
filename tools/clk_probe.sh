nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,power.limit,clocks_throttle_reasons.active --format=csv -lms 50 > gpurun_out/clk.csv 2>&1 &
SMI=$!
python tools/profile_step.py time > gpurun_out/clk_time.txt 2>&1
kill $SMI
tail -3 gpurun_out/clk_time.txt
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/clk.csv')))[1:]
vals=[(float(r[1].split()[0]), float(r[2].split()[0]), r[4].strip()) for r in rows if len(r)>4 and 'MHz' in r[1]]
busy=[v for v in vals if v[1]>300]
print(len(vals), 'samples;', len(busy), 'with power > 300 W')
if busy:
    import statistics as st
    print('sm MHz median', st.median(v[0] for v in busy), 'power W median', st.median(v[1] for v in busy), 'max', max(v[1] for v in busy))
    print(set(v[2] for v in busy))
PY
