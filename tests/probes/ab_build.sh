# Build the committed (HEAD) version of semd_eval.cu into libsemd_b200_ab.so for A/B runs
# against the working tree's libsemd_b200.so (select with SEMD_LIB).
set -e
cd "$(dirname "$0")/../../paper_2106_15319_b200/csrc"
python build.py > /dev/null
git show HEAD:paper_2106_15319_b200/csrc/${1:-semd_eval.cu} > /tmp/ab_src.cu
cp /tmp/ab_src.cu ./_ab_src.cu
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr"
$NV -c _ab_src.cu -o /tmp/ab.o
rm -f _ab_src.cu
objs=""
for f in semd_eval semd_sift semd_aux semd_resident semd_capi; do
  if [ "$f.cu" = "${1:-semd_eval.cu}" ]; then objs="$objs /tmp/ab.o"; else objs="$objs $f.o"; fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o ../libsemd_b200_ab.so $objs -lcudart
