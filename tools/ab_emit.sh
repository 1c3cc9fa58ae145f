#!/bin/bash
# A/B of the emit kernel: build HEAD~N vs working tree? (here: current tree only), 3 bench runs per CE
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for ce in ${CES:-1e-3 1e-2}; do for r in 1 2 3; do
  timeout 300 python bench.py --ce $ce --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ce', '$ce', 'emit %.2f' % d['kernel_ms_per_step']['emit'], 'frac %.3f' % d['roofline']['frac'], 'value %.4g' % d['value'])"
done; done
