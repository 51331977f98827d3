# build an experimental variant of libmgb200 into exp/lib_$1.so from a copy of the tree with a
# python patch applied: bash tools/ab/build.sh NAME patch.py   (output in exp/, git-ignored scratch)
set -e
mkdir -p exp
N=$1; PATCH=$2; D=/tmp/exp_$N
rm -rf $D; mkdir -p $D/b; cp -r paper_1406_5369_b200/csrc include $D/
[ -n "$PATCH" ] && python $PATCH $D/csrc
NC=/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl
for f in $D/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC,-O2 \
    -I $D/include -I $D/csrc -I $NC/include -c $f -o $D/b/$(basename $f .cu).o 2>&1 | grep -E ' error' &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/lib_$N.so $D/b/*.o -L $NC/lib -l:libnccl.so.2 -Xlinker -rpath,$NC/lib
echo "built exp/lib_$N.so"
