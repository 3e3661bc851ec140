# The whole GPU test suite against the range-checked build (-DPMX_CHECKED),
# then the zero-violation assertion (tests/test_zz_checked.py runs last).
set +e
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
[ -f build/variants/checked/libpmx_cuda.so ] || tools/variants.sh checked:"-DPMX_CHECKED" > /dev/null
PMX_LIB=$PWD/build/variants/checked/libpmx_cuda.so timeout 1800 python -m pytest tests -m gpu -q -rA \
  > gpurun_out/checked_tests.log 2>&1
echo "checked suite rc=$?"
grep -E "passed|failed|test_no_range_violations" gpurun_out/checked_tests.log | tail -4
