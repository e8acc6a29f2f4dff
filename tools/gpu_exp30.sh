for rep in 1 2; do
  for v in "-DNACCX_TEX_MINB=1" "-DNACCX_TEX_MINB=8"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    timeout 600 python bench.py --steps 100 --warmup 5 --no-extras --no-cpu-baseline > /tmp/b.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/b.json')); print('$v', 'ms', round(d['ms_per_step'],4), 'field_sigma', round(d['stage_ms']['field_sigma']*1e3,1))"
  done
done
