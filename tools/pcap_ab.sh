#!/bin/bash
# k_emit point-cache size A/B (LMM_PCAP override, PCAP_MIN + 16 k): emit ms per config
for c in ${CFGS:-octet100 bcc250}; do for p in "" ${PCAPS:-312}; do
  LMM_PCAP=$p timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pc.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pc.json').read().strip().splitlines()[-1]); print('$c', 'pcap=$p', 'value %.4g' % d['value'], 'emit %.2f' % d['kernel_ms_per_step']['emit'], 'frac %.4f' % d['roofline']['frac'])"
done; done
