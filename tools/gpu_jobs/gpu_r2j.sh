python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/j_build.log 2>&1
timeout 300 python tools/fft_probe.py 512 > gpurun_out/j_probe.log 2>&1
CGL_LIB_OVERRIDE=$PWD/tmp_ab/libgv1.so timeout 300 python tools/fft_probe.py 512 > gpurun_out/j_probe_gv1.log 2>&1
CGL_LIB_OVERRIDE=$PWD/tmp_ab/libgv2.so timeout 300 python tools/fft_probe.py 512 > gpurun_out/j_probe_gv2.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 2 --no-extras > gpurun_out/j_bench.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 2 --no-extras --scheme strang > gpurun_out/j_bench_strang.log 2>&1
head -14 gpurun_out/j_probe.log; grep "G axis" gpurun_out/j_probe_gv*.log; cut -c1-250 gpurun_out/j_bench.log gpurun_out/j_bench_strang.log
