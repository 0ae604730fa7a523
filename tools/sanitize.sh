# compute-sanitizer over tools/sanitize_run.py (run on a GPU box from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash tools/sanitize.sh'
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 99 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize_$tool.log
done
