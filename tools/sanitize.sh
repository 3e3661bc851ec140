# compute-sanitizer (one tool per gpurun call) over the GPU tests at small sizes.
# usage: bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
set +e
TOOL=${1:-memcheck}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
SEL='not shape1 and not match_and_refine_parity and not full_size and not 400'
timeout 2400 compute-sanitizer --tool $TOOL --error-exitcode 99 --print-limit 50 \
  python -m pytest tests/test_matching_gpu.py tests/test_tracking_gpu.py tests/test_backend_gpu.py \
  tests/test_exactness_gpu.py tests/test_golden.py tests/test_neighbours.py -m gpu -q -x -k "$SEL" \
  > gpurun_out/sanitizer_$TOOL.log 2>&1
echo "sanitizer $TOOL rc=$?"
grep -E "ERROR SUMMARY|passed|failed|Error" gpurun_out/sanitizer_$TOOL.log | tail -5
