#!/bin/bash
# Runs the reference's unit suites (built against the drop-in) + GPU pytest.
mkdir -p gpurun_out/rs
for t in tests/refsuite/_build/test_*; do
  n=$(basename $t)
  timeout 300 $t > gpurun_out/rs/$n.log 2>&1; echo "exit $?" >> gpurun_out/rs/$n.log
done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/rs/pytest.log 2>&1; echo "exit $?" >> gpurun_out/rs/pytest.log
