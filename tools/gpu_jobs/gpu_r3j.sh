timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tucker2d or C0 or baseline_config or stepper" > gpurun_out/j3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/j3_pytest.log
tail -n 4 gpurun_out/j3_pytest.log
for i in 1 2; do timeout 300 python tools/prof_step.py strang 200 C0; done
timeout 300 python tools/prof_step.py if4 200 C0
