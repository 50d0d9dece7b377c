for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2; done
timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "STR_|G axis" | grep -v "^{"
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/m3_bench.log 2>&1; cut -c1-260 gpurun_out/m3_bench.log
