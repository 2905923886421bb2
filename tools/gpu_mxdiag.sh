cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 python tools/mx_diag.py > gpurun_out/mx_diag.log 2>&1; echo rc=$? >> gpurun_out/mx_diag.log
