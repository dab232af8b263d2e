# Build A/B variants of the library into _variants/<name>/ (git-ignored; travels with gpurun).
#   bash scripts/build_variants.sh name1 "FLAGS1" name2 "FLAGS2" ...
set -e
cd "$(dirname "$0")/../paper_2205_03532_b200/csrc"
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  make -s -j8 OUT=../../_variants/$name/libcontactsim_b200.so OBJDIR=../../_variants/$name/obj EXTRA_NVFLAGS="$flags"
  echo "built $name ($flags)"
done
