# SpMV on the skewed matrices of spmv_skew.py under tuning overrides:
#   bash tools/micro/skew_sweep.sh "RLT_SPMV_LONG_PIECE=512 RLT_SPMV_LONG_GROUP=8" "RLT_SPMV_ROWS=4" ...
for cfg in "$@"; do
    echo "== $cfg"
    env $cfg python tools/micro/spmv_skew.py 2>&1 | grep case | sed "s/'nnz'.*'cc'/'cc'/; s/, 'relerr'.*//"
done
