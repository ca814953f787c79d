python -m pytest tests/test_gpu_parity.py -q -x -k "toeplitz" 2>&1 | tail -2
BEM_TZ_SHAPE=0 python -m pytest tests/test_gpu_parity.py -q -x -k "toeplitz" 2>&1 | tail -2
for sh in 0 1 2 1; do
BEM_TZ_SHAPE=$sh python bench.py --variant toeplitz --config C4 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('shape',$sh,d['ms_per_step'],d['roofline']['achieved'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done
for sh in 0 1; do
BEM_TZ_SHAPE=$sh python bench.py --variant toeplitz --config C3 --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('C3 shape',$sh,d['ms_per_step'],d['roofline']['achieved'],d['roofline']['frac'])"
done
