# Programmatic-dependent-launch A/B: device-resident steps and chunked (e2e-style) launches
# for SWEDG_PDL bit masks (1 modal volume, 2 modal interface, 4 SBP).
for m in 0 1 2 3; do
  echo "== SWEDG_PDL=$m"
  SWEDG_PDL=$m python tools/pdl_step_probe.py 1024 2>&1 | tail -3
  SWEDG_PDL=$m python tools/chunk_overhead.py 1024 2>&1 | grep "chunks  16"
done
