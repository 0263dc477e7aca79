# DRAM bytes / L2 hit rate of the fused kernel (C5) for several TY (tuning off)
mkdir -p gpurun_out
for ty in 4 6 8; do
  VX_FUSED_TY=$ty ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:k_step_fused -s 3 -c 2 --csv \
    python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --engine fused > gpurun_out/ncu_ty$ty.csv 2>/dev/null
  echo "TY=$ty"; grep -E "dram__bytes|hit_rate|duration" gpurun_out/ncu_ty$ty.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -8
done
