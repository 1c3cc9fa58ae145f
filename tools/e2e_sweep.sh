for F in "" "-DLMM_NSTAGE=3" "-DLMM_NSTAGE=4 -DLMM_STAGE_LOG2=21" "-DLMM_STAGE_LOG2=23"; do
  export LMM_NVCC_EXTRA="$F"
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  timeout 600 python bench.py --steps 1 --warmup 1 --e2e-steps 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "
import json; d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]); print('[$F]', 'e2e %.3g' % d['e2e']['value'], round(d['e2e']['ms_per_step']))"
done
python tools/d2h_bw.py
