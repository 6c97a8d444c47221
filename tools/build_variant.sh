#!/bin/bash
# Experiment helper: libbsgpu with some translation units rebuilt from a
# modified copy of csrc/ (the rest from build/).
# usage: tools/build_variant.sh <name> <variant csrc dir> <file.cu>... [-- extra nvcc flags]
# -> paper_2405_13943_b200/lib_var/libbsgpu_<name>.so (select with BSG_LIB=...)
set -e
NAME=$1; VDIR=$2; shift 2
FILES=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do FILES+=("$1"); shift; done
[ "${1:-}" = "--" ] && shift
D=/root/repo/paper_2405_13943_b200
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p $D/lib_var $D/build_var/$NAME
for f in "${FILES[@]}"; do
  FL="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I$D/../include"
  case $f in preprocess.cu|densify.cu) FL="$FL --fmad=false";; esac
  nvcc $FL "$@" -Xptxas -v -c $VDIR/$f -o $D/build_var/$NAME/${f%.cu}.o 2> $D/build_var/$NAME/${f%.cu}.ptxas.log || { cat $D/build_var/$NAME/${f%.cu}.ptxas.log; exit 1; }
done
OBJS=""
for o in $D/build/*.o; do
  b=$(basename $o .o)
  if [ -f $D/build_var/$NAME/$b.o ] && printf '%s\n' "${FILES[@]}" | grep -qx "$b.cu"; then OBJS="$OBJS $D/build_var/$NAME/$b.o"; else OBJS="$OBJS $o"; fi
done
nvcc $ARCH -shared -o $D/lib_var/libbsgpu_${NAME}.so $OBJS -ldl -lpthread
echo built $D/lib_var/libbsgpu_${NAME}.so
