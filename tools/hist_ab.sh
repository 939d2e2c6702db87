# The GEMM / NTT kernels of an earlier commit against HEAD, on the same box:
#   [CFGS="2 13 14"] bash tools/hist_ab.sh [COMMIT]   (default cbd8577, the round-2 state before the tile-run work)
# libqrng_<commit>.so is built from `git archive` of that commit's sources (needs
# the git metadata: build it here, it travels with the snapshot), loaded via QRNG_LIB_PATH.
C=${1:-cbd8577}
L=paper_2011_04130_b200/libqrng_$C.so
if [ ! -f $L ]; then
  d=$(mktemp -d); git archive $C paper_2011_04130_b200/csrc include | tar -x -C $d || exit 1
  for f in $d/paper_2011_04130_b200/csrc/*.cu; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo --expt-relaxed-constexpr -Xcompiler -fPIC \
         -Xcompiler -fvisibility=hidden -I $d/include -c $f -o ${f%.cu}.o & done; wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L $d/paper_2011_04130_b200/csrc/*.o -Xcompiler -fPIC || exit 1
  rm -rf $d
  [ -z "$GRAFT_REPO_ROOT" ] && { echo "built $L; run this script on the GPU box now"; exit 0; }
fi
python -m paper_2011_04130_b200.build > /dev/null || exit 1
for i in 1 2; do for lib in libqrng_$C.so libqrng.so; do for c in ${CFGS:-18 10 1 2 3 4}; do
  QRNG_LIB_PATH=$PWD/paper_2011_04130_b200/$lib python bench.py --config $c --configs none --no-e2e --no-cpu-baseline > gpurun_out/h.json 2>/dev/null; python tools/line.py "$lib cfg$c" < gpurun_out/h.json
done; done; done
