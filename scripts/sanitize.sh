# compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# scripts/sanitize_driver.py; logs to gpurun_out/ (summaries -> profiles/)
cd "$(dirname "$0")/.."
rm -f gpurun_out/r02_sanitize_rc.txt
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
    python scripts/sanitize_driver.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02_sanitize_rc.txt
done
