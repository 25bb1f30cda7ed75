# round 2, job bm: extended seeded sweep on the final code -- 8 further draws of the 96 random cases of
# tests/test_gpu_sweep.py::test_random_sweep (variants, shapes, spectra incl. gapped / rank-deficient), graded by tests/parity.py
: > gpurun_out/extended_sweep.txt
for off in 100000 200000 300000 400000 500000 600000 700000 800000; do
  echo "RQLP_SWEEP_OFFSET=$off" >> gpurun_out/extended_sweep.txt
  RQLP_SWEEP_OFFSET=$off timeout 900 python -m pytest tests/test_gpu_sweep.py -q -p no:cacheprovider -k test_random_sweep 2>&1 | tail -15 >> gpurun_out/extended_sweep.txt
done
echo done
