# MP step vs the streaming-grid wave count (MPX_STREAM_WAVES; "def" = the library's rule)
for i in 1 2; do for w in ${WAVES:-def 1 4 8 12}; do
  if [ "$w" = def ]; then unset MPX_STREAM_WAVES; else export MPX_STREAM_WAVES=$w; fi
  timeout -s KILL 300 python bench.py --steps 300 --warmup 10 --no-cpu-baseline --no-vit > gpurun_out/abw.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/abw.log').read().strip().splitlines()[-1]); print('waves $w', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['ms_per_step'], d['e2e']['value'])"
done; done
unset MPX_STREAM_WAVES
