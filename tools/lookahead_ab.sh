python -m paper_2011_04130_b200.build > /dev/null
python -m paper_2011_04130_b200.build --variant tl -DQRNG_GEMM_TIMELINE > /dev/null
for c in 2 3; do QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/libqrng_tl.so python tools/gemm_timeline.py --config $c; done

