timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sharded or slab" > gpurun_out/i3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/i3_pytest.log
tail -n 25 gpurun_out/i3_pytest.log
