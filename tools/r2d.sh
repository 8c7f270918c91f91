export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/checks
export ASR_LIB_PATH=$PWD/build/libasr_checks.so
timeout 900 python tools/sanitize.py > gpurun_out/checks/cases.log 2>&1; echo cases_rc=$?; tail -6 gpurun_out/checks/cases.log
