for i in 1 2; do for lib in paper_2507_03312_b200/lib/libmpx_b200.so abl/libmpx_g4.so; do
  MPX_B200_LIB=$PWD/$lib timeout -s KILL 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-vit > gpurun_out/abmp.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/abmp.log').read().strip().splitlines()[-1]); print('$lib', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['ms_per_step'])"
done; done
