# A/B of the iris match kernel variants (alternating processes, same box):
# default build, build/variants/libirl_noslots.so (-DIRL_SPLIT_SLOTS=0),
# build/variants/libirl_head.so (the previous commit's kernel)
set -x
timeout 900 python -m pytest tests/test_iris.py tests/test_fold.py -m gpu -x -q 2>&1 | tail -3
python profiles/iris_diag.py --runs 1
IRL_B200_LIB=build/variants/libirl_head.so python profiles/iris_diag.py --runs 1
for i in 1 2 3; do
  python profiles/iris_match_ab.py --reps 30
  IRL_B200_LIB=build/variants/libirl_noslots.so python profiles/iris_match_ab.py --reps 30
  IRL_B200_LIB=build/variants/libirl_head.so python profiles/iris_match_ab.py --reps 30
done
IRL_IRIS_I8=1 python profiles/iris_match_ab.py --reps 30
IRL_IRIS_I8=1 IRL_B200_LIB=build/variants/libirl_head.so python profiles/iris_match_ab.py --reps 30
