python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/m_build.log 2>&1


timeout 1500 python tools/project_sharded.py 1 2 4 8 --steps 3 > gpurun_out/m_project.log 2>&1; echo "rc=$?" >> gpurun_out/m_project.log
tail -n 5 gpurun_out/m_pytest.log gpurun_out/m_pytest_fft.log; cat gpurun_out/m_project.log | tail -8
