# GPU test suite + smoke (no -x: report every failure).  Usage: bash tools/gpu_tests.sh <tag> [pytest args]
TAG=${1:-t}; shift
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider -rf "$@" > gpurun_out/pytest_$TAG.log 2>&1; tail -15 gpurun_out/pytest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
