# Iris match with the query on M (4x1 clusters, one pass) vs the database on M
# (1x4 clusters + a 32-column remainder pass, IRL_IRIS_DB_ON_M=1): same build,
# alternating processes on one box.
set -x
timeout 900 python -m pytest tests/test_iris.py tests/test_fold.py -m gpu -x -q 2>&1 | tail -3
python profiles/iris_diag.py --runs 1
for i in 1 2 3; do
  python profiles/iris_match_ab.py --reps 30
  IRL_IRIS_DB_ON_M=1 python profiles/iris_match_ab.py --reps 30
done
