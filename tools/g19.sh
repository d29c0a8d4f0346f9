set -u
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py --cfg 1 4 --balance > gpurun_out/san/$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san/$tool.log
done
