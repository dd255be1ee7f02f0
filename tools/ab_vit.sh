# same-box A/B of the ViT-B/16 training step: abl/ref_tree (a committed revision) vs the working tree
for t in abl/ref_tree . abl/ref_tree .; do
  (cd $t && timeout -s KILL 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /tmp/ab.log 2>&1)
  python -c "
import json; d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]); v=d['vit_b16_train']; print('$t', v['value'], v['ms_per_step'], d['clocks']['sm_mhz'])"
done
