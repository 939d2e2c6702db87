# Q-buffer kernel launch shape at deep trees (config 3, 2^17) and config 2
python -m paper_2011_04130_b200.build > /dev/null
python -m paper_2011_04130_b200.build --variant qd592 -DQRNG_QBUF_DIV=592 > /dev/null
python -m paper_2011_04130_b200.build --variant qd1184 -DQRNG_QBUF_DIV=1184 > /dev/null
python -m paper_2011_04130_b200.build --variant qu8 -DQRNG_QBUF_U=8 > /dev/null
for lib in libqrng.so libqrng_qd592.so libqrng_qd1184.so libqrng_qu8.so; do for c in 2 3 17; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/q.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/q.json
done; done
