mkdir -p gpurun_out/cli
export LSHBEAM_CLI=$PWD/paper_1806_00588_b200/lshbeam
cd tests/refsuite/_build
timeout 900 ./test_cli > ../../../gpurun_out/cli/test_cli.log 2>&1; echo "exit $?" >> ../../../gpurun_out/cli/test_cli.log
timeout 1500 ./acceptance $LSHBEAM_CLI > ../../../gpurun_out/cli/acceptance.log 2>&1; echo "exit $?" >> ../../../gpurun_out/cli/acceptance.log
