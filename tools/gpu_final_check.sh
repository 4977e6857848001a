timeout 300 python __graft_entry__.py --smoke; echo smoke_rc=$?
timeout 900 python -m pytest tests/test_gpu_contract.py tests/test_gpu_factorize.py tests/test_gpu_gemm_shapes.py tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-near-kernel --steps 3 --warmup 3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['n_cg'], d['gemm']['tflops'])"
