run() { CHGPU_NO_JOIN=$2 python scripts/sweep.py --points 8192 --shapes uniform sift --no-guided | python -c "
import sys,json
print('RESULT $1', [round(json.loads(l)['pairs_per_s_kernel']) for l in sys.stdin])"; }
run adaptive_nojoin 1
run adaptive_join 0
