# build libns2b.so variants here (name=flags ...) into _variants/<name>.so; the default build last
set -e
for spec in "$@"; do name=${spec%%=*}; flags=${spec#*=}
  NS2B_NVCC_EXTRA="$flags" python -m paper_2212_05231_b200.build --force > /dev/null
  cp paper_2212_05231_b200/libns2b.so _variants/$name.so; echo "built $name ($flags)"
done
python -m paper_2212_05231_b200.build --force > /dev/null; cp paper_2212_05231_b200/libns2b.so _variants/base.so
