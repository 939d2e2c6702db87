python -m paper_2011_04130_b200.build > /dev/null
for c in 2 4 8; do python -m paper_2011_04130_b200.build --variant h$c -DQRNG_HIST_COPIES=$c > /dev/null; done
for lib in libqrng.so libqrng_h2.so libqrng_h4.so libqrng_h8.so; do echo $lib; QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python tools/bench_minentropy.py; done
