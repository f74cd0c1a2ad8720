# A/B launch-shape knobs on one workload (GPU box): bash tools/ab_env.sh <workload> "ENV=.. ENV=.." ...
W=$1; shift
for cfg in "$@"; do
  env $cfg python bench.py --steps 30 --warmup 5 --workload $W --no-cpu --no-variants 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', round(d['value']), 'us/step', round(d['us_per_step'],1), 'attn_us', round(r['launch_ms']*1e3,1), 'frac', round(r['frac'],3))"
done
