# GPU tests + the reference's own test suite against the package (levlu alias)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
ROOTD=$(pwd)
mkdir -p gpurun_out
TAG=${TAG:-r2}
timeout -s ABRT 1200 python -X faulthandler -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest gpu rc=$?"; tail -4 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
if [ -d baseline/_ref/tests ]; then
  (cd baseline/_ref/tests && PYTHONPATH=$ROOTD/tools/levlu_alias:$ROOTD timeout 1200 python -m pytest -q -p no:cacheprovider -rfEs . > $ROOTD/gpurun_out/ref_suite_${TAG}.log 2>&1; echo "ref suite rc=$?")
  tail -15 gpurun_out/ref_suite_${TAG}.log
fi
