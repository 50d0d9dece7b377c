python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/o_build.log 2>&1
CGL_FULLRUN_LOG=gpurun_out/o_fullruns.jsonl timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/o_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/o_pytest.log
timeout 300 python tools/prof_step.py strang 200 C0 > gpurun_out/o_c0.log 2>&1
CGL_TUCKER2D=0 timeout 300 python tools/prof_step.py strang 200 C0 >> gpurun_out/o_c0.log 2>&1
timeout 300 python tools/prof_step.py if4 200 C0 >> gpurun_out/o_c0.log 2>&1
CGL_TUCKER2D=0 timeout 300 python tools/prof_step.py if4 200 C0 >> gpurun_out/o_c0.log 2>&1
tail -n 8 gpurun_out/o_pytest.log; cat gpurun_out/o_c0.log; cat gpurun_out/o_fullruns.jsonl
