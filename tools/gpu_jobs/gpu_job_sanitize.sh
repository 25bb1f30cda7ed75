# compute-sanitizer memcheck (then racecheck / synccheck) on C1 and C2 through tools/run_one.py:
# eager first call, graph capture + replay on the later ones; plus the loopback ranks and the host feed
TOOL=${1:-memcheck}
for args in "--workload c1 --reps 3" "--workload c1e --reps 3" "--workload c2 --reps 3" "--workload c1 --reps 2 --loopback 3" "--workload c1e --reps 2 --host"; do
  tag=$(echo $args | tr -d ' -' )
  timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python tools/run_one.py $args > gpurun_out/san_${TOOL}_${tag}.log 2>&1
  echo "$TOOL $args rc=$?"; tail -3 gpurun_out/san_${TOOL}_${tag}.log
done
