cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 120 python tools/fit_once.py c4 1000 3 2>&1 | tail -n 2; }
{
run AIWC_X=0
run AIWC_WIDE_LANES=3
run AIWC_WIDE_LANES=5
run AIWC_WIDE_PER_SM=3
run AIWC_WIDE_PER_SM=5
run AIWC_BIG_MIN=2048
run AIWC_BIG_MIN=8192
run AIWC_LANE_MAX=8
run AIWC_LANE_MAX=32
} > gpurun_out/sweep.log 2>&1
