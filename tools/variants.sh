# Build ablation variants of libpmx_cuda.so into build/variants/<name>/ (dev tool).
# usage: tools/variants.sh name1:"-DPMX_PRUNE=0" name2:"-DPMX_LD256=0 -DPMX_RCP=0" ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  out=$ROOT/build/variants/$name
  mkdir -p $out
  cp $ROOT/paper_2412_12392_b200/csrc/*.cu $ROOT/paper_2412_12392_b200/csrc/*.cuh $ROOT/paper_2412_12392_b200/csrc/Makefile $out/
  mkdir -p $ROOT/build/include && cp $ROOT/include/pmx.h $ROOT/build/include/
  (cd $out && sed -i "s#../../include/pmx.h#$ROOT/include/pmx.h#" Makefile && \
   make -s -j6 NVCCFLAGS="-O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -I$ROOT/paper_2412_12392_b200/csrc $defs" >/dev/null)
  echo "$name: $(grep -A2 "Compiling entry function '_ZN3pmx14k_match_refine" $out/match.ptxas.log | tail -1)"
done
