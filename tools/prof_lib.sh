# profile one library variant's fused kernel (fixed geometry): bash /tmp/prof_lib.sh lib tag TY SX
cp paper_1212_2845_b200/libvoxsim.so /tmp/lib_orig.so
cp $1 paper_1212_2845_b200/libvoxsim.so
VX_FUSED_TY=$3 VX_FUSED_SX=$4 ncu --set full --import-source on --clock-control base -k regex:k_step_fused -s 20 -c 1 -o gpurun_out/prof_$2 python tools/ab_time.py x > gpurun_out/prof_$2.log 2>&1
echo rc=$?
cp /tmp/lib_orig.so paper_1212_2845_b200/libvoxsim.so
