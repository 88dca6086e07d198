# A/B of the far kernel's minimum CTAs per SM (register cap): rebuild, bench
for mb in ${MBS:-5 6 4}; do
  touch paper_2203_11733_b200/csrc/gbem_assembly.cu
  GBEM_NVCC_EXTRA="-DGBEM_FAR_MINB=$mb" python -c "from paper_2203_11733_b200 import build as b; b.build()" > /dev/null 2>&1 || echo "build $mb failed"
  echo "minb=$mb"; bash tools/far_ab.sh
done
