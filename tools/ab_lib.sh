# A/B two builds of libmpx_b200.so on the same box: abl/libmpx_head.so vs the working tree's
for lib in abl/libmpx_head.so paper_2507_03312_b200/lib/libmpx_b200.so abl/libmpx_head.so paper_2507_03312_b200/lib/libmpx_b200.so; do
  export MPX_B200_LIB=$PWD/$lib
  timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); v=d['vit_b16_train']; print('$lib', v['value'], v['ms_per_step'], d['clocks']['sm_mhz'])"
  python tools/time_gemm_modes.py
done
