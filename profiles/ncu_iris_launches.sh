ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/iris_launches.csv python profiles/iris_match_ab.py --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/iris_launches.csv')))
hdr=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
h=rows[hdr]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[hdr+1:][-12:]:
    print(r[ki][:90], r[vi])
PY
