python -m paper_2011_04130_b200.build > /dev/null || exit 1

python tools/oneshot_jitter.py --config 4 --steps 100 | tee gpurun_out/jitter_r2b.txt
python tools/oneshot_jitter.py --config 4 --steps 100 --flush 0 | tee -a gpurun_out/jitter_r2b.txt
python tools/oneshot_jitter.py --config 2 --steps 200 | tee -a gpurun_out/jitter_r2b.txt
python tools/small_batch.py > gpurun_out/small_narrow.txt
QRNG_GEMM_NARROW=0 python tools/small_batch.py > gpurun_out/small_wide.txt

