# same-box A/B of the ViT step with PDL on every launch (MPX_PDL_ALL=1) vs the MP-step chain only
for i in 1 2; do for v in 0 1; do
  MPX_PDL_ALL=$v timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --vit-steps 20 > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); v=d['vit_b16_train']; print('PDL_ALL=$v', v['value'], v['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
