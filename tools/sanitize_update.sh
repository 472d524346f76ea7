# compute-sanitizer racecheck + synccheck + memcheck on the update kernel over short runs (1 GPU)
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python tools/race_update.py 300 > gpurun_out/racecheck_update.log 2>&1; echo "racecheck update rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/race_update.py 300 > gpurun_out/synccheck_update.log 2>&1; echo "synccheck update rc=$?"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/race_update.py 600 > gpurun_out/memcheck_update.log 2>&1; echo "memcheck update rc=$?"
for f in gpurun_out/racecheck_update.log gpurun_out/synccheck_update.log gpurun_out/memcheck_update.log; do echo "== $f"; tail -n 5 $f; done
