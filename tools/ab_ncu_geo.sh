# A/B of (library, TY, SX) triples by ncu kernel duration at locked base clocks:
#   bash tools/ab_ncu_geo.sh lib.so:4:16 lib2.so:4:-1 ...   (SX < 0: ranged split, -SX waves)
mkdir -p gpurun_out
cp paper_1212_2845_b200/libvoxsim.so /tmp/lib_orig.so
for pass in ${PASSES:-1 2}; do
  for spec in "$@"; do
    IFS=: read lib ty sx <<< "$spec"
    cp $lib paper_1212_2845_b200/libvoxsim.so
    VX_FUSED_TY=$ty VX_FUSED_SX=$sx timeout 600 ncu --metrics gpu__time_duration.sum --clock-control base \
      -k regex:k_step_fused -s 20 -c ${NCNT:-15} --csv python tools/ab_time.py x > /tmp/ab_ncu.csv 2>/dev/null
    python - "$spec" <<'PY'
import csv, sys, statistics
rows = [r for r in csv.reader(open("/tmp/ab_ncu.csv")) if len(r) > 10]
hdr = next(r for r in rows if "Metric Value" in r)
iv = hdr.index("Metric Value")
vals = [float(r[iv].replace(",", "")) for r in rows if r is not hdr and r[iv] != "Metric Value"]
print(f"{sys.argv[1]:28s} median {statistics.median(vals) / 1e6:.4f} ms, min {min(vals) / 1e6:.4f} (n={len(vals)}) at base clocks")
PY
  done
done
cp /tmp/lib_orig.so paper_1212_2845_b200/libvoxsim.so
