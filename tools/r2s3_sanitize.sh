set -u
mkdir -p gpurun_out
which compute-sanitizer > gpurun_out/s3z_sanitizers_full.txt 2>&1
for t in memcheck racecheck initcheck; do echo "== $t" >> gpurun_out/s3z_sanitizers_full.txt; timeout 900 compute-sanitizer --tool $t python tools/sanitize.py >> gpurun_out/s3z_sanitizers_full.txt 2>&1; echo "exit $?" >> gpurun_out/s3z_sanitizers_full.txt; done
grep -E "COMPUTE-SANITIZER|SUMMARY|sanitize cases|^== |exit" gpurun_out/s3z_sanitizers_full.txt > gpurun_out/s3z_sanitizers.txt
echo done
