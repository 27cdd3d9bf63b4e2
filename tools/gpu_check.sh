# GPU-box helper: parity tests of the current build, then A/B kernel timing of in-tree variants.
# usage (via gpurun): bash tools/gpu_check.sh <tag> [variant.so ...]
tag=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/${tag}_gpu_tests.log
timeout 600 python tools/ab_time.py 3 40 libntbc.so "$@" > gpurun_out/${tag}_ab.log 2>&1
