#!/bin/bash
# deferred-pass CTA cap sweep (bench line per setting)
mkdir -p gpurun_out
for c in 1 2 4; do
  CH_STAGED_FB_CTAS=$c timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --locality staged > gpurun_out/fb_$c.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/fb_$c.json'));print($c, round(d['value'],3), d['phase_ms'])"
done
