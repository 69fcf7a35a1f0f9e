#!/bin/bash
mkdir -p gpurun_out/acc
cd tests/refsuite/_build && timeout 1800 ./acceptance /nonexistent/lshbeam_cli > ../../../gpurun_out/acc/acceptance.log 2>&1; echo "exit $?" >> ../../../gpurun_out/acc/acceptance.log
