mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  SANITIZE_TOOL=$tool timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|sanitize case|Error|error" gpurun_out/sanitize_$tool.txt | head -5
done
