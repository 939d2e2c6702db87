# NTT multi-pass: segment inputs from the raw bits (SEGBITS) vs the forward global passes
python -m paper_2011_04130_b200.build > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_modified.py tests/test_gpu_sweep.py -q -x -k "multipass or config_full_size or sweep or max_seed or modified or config4b or random" 2>&1 | tail -2
for v in 1 0; do for c in 4 19 22 17; do
  QRNG_NTT_BITS_PROLOGUE=$v python bench.py --config $c --path ntt --configs none --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python tools/line.py "bits=$v cfg$c"
done; done
QRNG_NTT_BITS_PROLOGUE=1 python bench.py --config 4 --variant modified --configs none --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python tools/line.py "bits=1 mod4"
QRNG_NTT_BITS_PROLOGUE=0 python bench.py --config 4 --variant modified --configs none --no-e2e --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python tools/line.py "bits=0 mod4"
