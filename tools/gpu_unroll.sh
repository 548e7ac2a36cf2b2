# row-group loop unroll sweep (modifies the box's scratch copy only)
for U in 1 2 4; do
  sed -i "s/^ *#pragma unroll [0-9]$/    #pragma unroll $U/" paper_1708_04174_b200/csrc/tridiag.cuh
  grep -c "pragma unroll $U\$" paper_1708_04174_b200/csrc/tridiag.cuh > gpurun_out/unroll_$U.log
  python -c "from paper_1708_04174_b200.build import build; build(force=True)" > gpurun_out/build_u$U.log 2>&1
  timeout 120 python tools/trd_prof.py 861 >> gpurun_out/unroll_$U.log 2>&1
done
