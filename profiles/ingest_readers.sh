# f3 ingest: parallel pread readers per 256 MB chunk (IRL_INGEST_READERS), one 18.5 GB part
python profiles/ingest_bench.py --keep > gpurun_out/ingest_write.json
F=$(python -c "import json; print(json.load(open('gpurun_out/ingest_write.json'))['file'])")
nproc
for r in 4 8 16 4 8 16; do IRL_INGEST_READERS=$r python profiles/ingest_bench.py --file $F; done
rm -f $F
