# A/B timing of abtest/* variants (tools/ab_run.sh), then the GPU tests with
# the variant named in $1 copied over the regular library.
mkdir -p gpurun_out
bash tools/ab_run.sh > gpurun_out/ab.log 2>&1; echo ab rc $?
cat gpurun_out/ab.log
if [ -n "$1" ]; then
  cp abtest/$1/librfd.so paper_2302_00942_b200/lib/librfd.so
  timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ab_tests.log 2>&1; echo tests rc $?
  tail -3 gpurun_out/ab_tests.log
fi
