# SIFT-shaped data: do the shortcuts pay?  (kernel-only pairs/s, 64 images x 8,192 points, join off)
run() { CHGPU_NO_JOIN=1 python scripts/sweep.py --points 8192 --shapes uniform sift --no-guided | python -c "
import sys,json
print('RESULT $1', [round(json.loads(l)['pairs_per_s_kernel']) for l in sys.stdin])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run base
b "-DCHGPU_NO_RERANK_SHORTCUT"; run no_rerank
b "-DCHGPU_NO_VERIFY_SHORTCUT -DCHGPU_NO_RERANK_SHORTCUT"; run no_shortcuts
b "-DCHGPU_NO_VERIFY_SHORTCUT"; run no_verify_shortcut
b ""
