# A/B of libvoxsim builds by ncu kernel durations at locked base clocks (stable
# under the power cap; fixed geometry TY=4 SX=16): bash tools/ab_ncu.sh a.so b.so ...
mkdir -p gpurun_out
cp paper_1212_2845_b200/libvoxsim.so /tmp/lib_orig.so
for pass in 1 2; do
  for lib in "$@"; do
    cp $lib paper_1212_2845_b200/libvoxsim.so
    VX_FUSED_TY=${TY:-4} VX_FUSED_SX=${SX:-16} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control base \
      -k regex:k_step_fused -s 20 -c 15 --csv python tools/ab_time.py $(basename $lib) > /tmp/ab_ncu.csv 2>/dev/null
    python - "$lib" <<'PY'
import csv, sys, statistics
rows = [r for r in csv.reader(open("/tmp/ab_ncu.csv")) if len(r) > 10]
hdr = next(r for r in rows if "Metric Value" in r)
iv = hdr.index("Metric Value"); iu = hdr.index("Metric Unit")
vals = []
for r in rows:
    if r is hdr or r[iv] == "Metric Value": continue
    v = float(r[iv].replace(",", "")); u = r[iu]
    vals.append(v * {"msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3}.get(u, 1.0))
print(f"{sys.argv[1]}: median {statistics.median(vals):.1f} us, min {min(vals):.1f} (n={len(vals)}) at base clocks")
PY
  done
done
cp /tmp/lib_orig.so paper_1212_2845_b200/libvoxsim.so
