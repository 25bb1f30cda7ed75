# round 2, job bh: parity calibration log of the whole -m gpu suite on the final code
rm -f gpurun_out/parity_log.jsonl
RQLP_PARITY_LOG=$PWD/gpurun_out/parity_log.jsonl timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_r2bh.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_r2bh.log
python tools/parity_calibration.py gpurun_out/parity_log.jsonl gpurun_out/r02_parity_calibration.json > gpurun_out/parity_calibration_summary.txt 2>&1
echo done
