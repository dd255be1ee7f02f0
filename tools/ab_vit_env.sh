for i in 1 2; do for cfg in "MPX_WGRAD_WIDE=0 MPX_B200_LIB=$PWD/abl/libmpx_head.so" "MPX_WGRAD_WIDE=1"; do
  env $cfg timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --vit-steps 20 > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); v=d['vit_b16_train']; print('$cfg'[:40], v['value'], v['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
