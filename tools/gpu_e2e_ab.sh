cd $GRAFT_REPO_ROOT
for o in 0 1 0 1; do
  APMG_SETUP_VOLFIRST=$o timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-inference --no-render 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print('volfirst=$o', round(d['value']/1e6,1), 'e2e', round(e['value']/1e6,1), e['setup_split_ms'], e['loop_ms'], e['wall_ms'])"
done
