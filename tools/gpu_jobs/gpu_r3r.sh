python -c "
from paper_2403_02816_b200 import _build
_build.build()
_build.build(out=_build.LIB_DIR + '/libtw3.so', extra_flags=('-DCGL_TW3',))" > gpurun_out/r3_build.log 2>&1
for i in 1 2; do
echo "default"; timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "plain|IF4_B1|IF4_B4" | grep -v "^{"
echo "TW3"; CGL_LIB_OVERRIDE=paper_2403_02816_b200/_lib/libtw3.so timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "plain|IF4_B1|IF4_B4" | grep -v "^{"
done
CGL_LIB_OVERRIDE=paper_2403_02816_b200/_lib/libtw3.so timeout 600 python -m pytest tests/test_fftpass.py -m gpu -x -q 2>&1 | tail -2
