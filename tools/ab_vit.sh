# same-box A/B of the ViT-B/16 training step: abl/ref_tree (a committed revision) vs the working tree
# usage: bash tools/ab_vit.sh [rounds] [vit steps]
R=${1:-2}; S=${2:-10}
for i in $(seq $R); do for t in abl/ref_tree .; do
  (cd $t && timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --vit-steps $S > /tmp/ab.log 2>&1)
  python -c "
import json; d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]); v=d['vit_b16_train']; print('$t', v['value'], v['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
