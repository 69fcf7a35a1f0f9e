mkdir -p gpurun_out/dbg
for i in 1 2; do
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/dbg/full_$i.log 2>&1; echo "exit $?" >> gpurun_out/dbg/full_$i.log
done
LSB_NO_X2=1 timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/dbg/nox2.log 2>&1; echo "exit $?" >> gpurun_out/dbg/nox2.log
