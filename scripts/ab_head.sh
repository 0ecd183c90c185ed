# usage: ab_head.sh "label|ENV|args" ...
for spec in "$@"; do
  label="${spec%%|*}"; rest="${spec#*|}"; envs="${rest%%|*}"; args="${rest#*|}"
  env $envs python bench.py --no-secondaries --no-e2e --no-zslab --no-cpu-baseline $args 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; o=r['other_kernel']
print('$label', round(d['value']), r['kernel'], round(r['avg_launch_us'],1), round(r['frac'],3), o['kernel'], round(o['avg_launch_us'],1), round(o['frac'],3))"
done
