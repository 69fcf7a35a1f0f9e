#!/bin/bash
mkdir -p gpurun_out/q2
timeout 600 python -m pytest tests/test_gpu_vocab_shard.py tests/test_gpu_stages.py -x -q --timeout 300 > gpurun_out/q2/pytest.log 2>&1; echo "exit $?" >> gpurun_out/q2/pytest.log
cd tests/refsuite/_build && timeout 1500 ./acceptance /nonexistent/lshbeam_cli > ../../../gpurun_out/q2/acceptance.log 2>&1; echo "exit $?" >> ../../../gpurun_out/q2/acceptance.log
