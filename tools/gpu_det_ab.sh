cd $GRAFT_REPO_ROOT
for r in 1 2; do for lib in "" "$PWD/ab/base/libapmg_cuda.so"; do
APMG_DETERMINISTIC=1 APMG_LIB="$lib" timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-inference --no-render --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('DET lib=${lib##*/ab/}', round(d['value']/1e6,1), round(d['roofline']['ms_per_launch'],4), d['final_l_rec'])"
done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "determin or multirank" 2>&1 | tail -1
