# Jacobi sweep counts per call (debug build of the library, in the box's scratch copy only)
python - <<'PY' > gpurun_out/jdbg_build.log 2>&1
import paper_1708_04174_b200.build as b
b.NVCC_FLAGS.append("-DSOSADMM_JACOBI_DEBUG")
print(b.build(force=True))
PY
timeout 300 python tools/jdbg.py > gpurun_out/jdbg.log 2>&1; echo jdbg=$?
