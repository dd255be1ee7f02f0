# same-box A/B of the ViT-B/16 training step under environment settings
# usage: bash tools/ab_env.sh ROUNDS "ENV_A" "ENV_B" ...   (e.g. "MPX_ATTN_PSAVE=1" "MPX_ATTN_PSAVE=0")
R=$1; shift
for i in $(seq $R); do for cfg in "$@"; do
  env $cfg timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-vit-l --no-second-half \
    --vit-steps 20 > gpurun_out/ab.log 2> gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); v=d['vit_b16_train']; print('$cfg'[:60], v['value'], v['ms_per_step'], d['clocks']['sm_mhz'], v.get('final_loss'))" || tail -5 gpurun_out/ab.err
done; done
