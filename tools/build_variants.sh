# build libburst variants of one kernel TU with extra -D flags: tools/build_variants.sh <tu> <name>:<flags> ...
set -e
TU=$1; shift
OBJ=paper_2509_19836_b200/_lib/obj
mkdir -p paper_2509_19836_b200/_lib/variants
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -Iinclude $flags -c paper_2509_19836_b200/csrc/$TU.cu -o /tmp/v_$name.o
  objs=$(ls $OBJ/*.o | grep -v "/$TU.o")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o paper_2509_19836_b200/_lib/variants/lib_$name.so $objs /tmp/v_$name.o
  echo built $name
done
