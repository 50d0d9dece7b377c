# round-2 check: GPU tests, bench (C3 headline), reference arm, 2-rank spawn path
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; free -g
python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/a_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/a_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/a_bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/a_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/a_ref.log
tail -n 3 gpurun_out/a_pytest.log gpurun_out/a_bench.log gpurun_out/a_ref.log
