# A/B of libvoxsim build variants on C5: bash tools/ab_libs.sh v1.so v2.so ...  (2 passes)
mkdir -p gpurun_out
cp paper_1212_2845_b200/libvoxsim.so /tmp/lib_orig.so
for pass in 1 2; do
  for lib in "$@"; do
    cp $lib paper_1212_2845_b200/libvoxsim.so
    VX_FUSED_TUNE_LOG=1 timeout 300 python tools/ab_time.py $(basename $lib) 2>&1 | grep -v "^$" | tail -2
  done
done
cp /tmp/lib_orig.so paper_1212_2845_b200/libvoxsim.so
