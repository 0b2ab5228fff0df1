cd $GRAFT_REPO_ROOT
for r in 1 2; do for lib in "" "$PWD/ab/ibase/libapmg_cuda.so"; do
APMG_LIB="$lib" timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('lib=${lib##*/ab/}', round(d['inference']['value']/1e9,3), 'Gvox/s', d['inference']['ms_per_sweep'], 'render', d['render'].get('ms_per_frame'))"
done; done
timeout 900 python -m pytest tests -m gpu -q -x -k "lattice or sweep or render or forward or infer or decomposed" 2>&1 | tail -1
