python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/a3_build.log 2>&1
python -c "
from paper_2403_02816_b200 import _build
_build.build(out=_build.LIB_DIR + '/libvar3.so', extra_flags=('-DCGL_R32_MINB=3',))" >> gpurun_out/a3_build.log 2>&1
for i in 1 2; do
echo "MINB=2"; timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "G axis" | grep -v "^{"
echo "MINB=3"; CGL_LIB_OVERRIDE=paper_2403_02816_b200/_lib/libvar3.so timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "G axis" | grep -v "^{"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_r32" -c 2 -o gpurun_out/a3_r32_full python tools/fft_probe.py 512 --ncu > gpurun_out/a3_ncu.log 2>&1
ncu -i gpurun_out/a3_r32_full.ncu-rep --page raw --csv > gpurun_out/a3_r32_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/a3_r32_raw.csv
