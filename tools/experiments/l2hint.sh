#!/bin/bash
# A/B of a build variant: HOPM rate + cfg2 bench headline (no components)
python tools/experiments/hopm_rate.py
python tools/experiments/hopm_rate.py
python bench.py --no-components --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg2', d['value'], d['roofline']['mean_launch_us'])"
