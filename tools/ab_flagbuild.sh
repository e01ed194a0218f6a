# Build libigs_b200.so variants of the working tree with extra nvcc flags for an A/B run:
#   bash tools/ab_flagbuild.sh NAME "-DFOO=1 -DBAR=2" [NAME2 "flags2" ...]  ->  ab/NAME/libigs_b200.so
# (HEAD is built as ab/HEAD when given the name HEAD with flags "").
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  mkdir -p ab/$name /tmp/abb_$name
  if [ "$name" = HEAD ]; then
    rm -rf /tmp/abb_HEAD && mkdir -p /tmp/abb_HEAD && git archive HEAD | tar -x -C /tmp/abb_HEAD
    src=/tmp/abb_HEAD/paper_2603_08661_b200/csrc
  else
    src=paper_2603_08661_b200/csrc
  fi
  objs=""
  for f in $src/*.cu; do
    o=/tmp/abb_$name/$(basename $f .cu).o
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false \
      -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -c $f -o $o &
    objs="$objs $o"
  done
  wait
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/$name/libigs_b200.so $objs
  echo "built ab/$name ($flags)"
done
