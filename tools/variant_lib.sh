#!/bin/bash
# Build an A/B variant of libigs_b200.so: tools/variant_lib.sh OUT.so SRC.cu "-DMACRO=V ..."
# (the other objects as built in _build/; load it with IGS_B200_LIB=OUT.so)
set -e
cd "$(dirname "$0")/.."
out=$1; src=$2; defs=$3
python -c "import __graft_entry__ as g; g.build()"
tmp=$(mktemp -d)
stem=$(basename "$src" .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-O2 \
  -I include --expt-relaxed-constexpr $defs -c "$src" -o "$tmp/$stem.o"
objs=$(ls paper_2407_01866_b200/_build/*.o | grep -v "/$stem.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs "$tmp/$stem.o" --cudart static -ldl
rm -rf "$tmp"
