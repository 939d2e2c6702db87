# Q-buffer kernel launch shape: blocks-per-CTA cap (QRNG_QBUF_MAXBPC, default 32), units in flight (QRNG_QBUF_U)
python -m paper_2011_04130_b200.build > /dev/null
python -m paper_2011_04130_b200.build --variant qb64 -DQRNG_QBUF_MAXBPC=64 > /dev/null
python -m paper_2011_04130_b200.build --variant qb128 -DQRNG_QBUF_MAXBPC=128 > /dev/null
python -m paper_2011_04130_b200.build --variant qb64u8 -DQRNG_QBUF_MAXBPC=64 -DQRNG_QBUF_U=8 > /dev/null
python -m paper_2011_04130_b200.build --variant qu8 -DQRNG_QBUF_U=8 > /dev/null
for i in 1 2; do for lib in libqrng.so libqrng_qb64.so libqrng_qb128.so libqrng_qb64u8.so libqrng_qu8.so; do for c in 2 3 13 17; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/q.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/q.json
done; done; done
