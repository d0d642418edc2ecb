cat > /tmp/run_bench_fh.py <<'PY'
import faulthandler, signal, sys, runpy
faulthandler.register(signal.SIGTERM, all_threads=True)
sys.argv = ["bench.py", "--steps", "20", "--warmup", "5", "--cpu-seconds", "0", "--no-bert", "--no-reducer"]
runpy.run_path("bench.py", run_name="__main__")
PY
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_dbg.csv timeout -s TERM 150 python /tmp/run_bench_fh.py > gpurun_out/ncu_dbg.out 2>&1; echo rc=$?
env | grep -i -E "inject|nsight|compute_prof" | head
tail -60 gpurun_out/ncu_dbg.out
