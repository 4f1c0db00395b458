# fold kernel A/B: default build vs build/variants/libirl_fold0.so (-DIRL_FOLD_PREFETCH=0), alternating
timeout 600 python -m pytest tests/test_fold.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do
  python profiles/fold_bench.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefetch', d['fold_kernel']['ms'])"
  IRL_B200_LIB=build/variants/libirl_fold0.so python profiles/fold_bench.py | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('r07loop ', d['fold_kernel']['ms'])"
done
