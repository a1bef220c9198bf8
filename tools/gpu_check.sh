set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g1_build.log 2>&1 || { echo build failed; tail gpurun_out/g1_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/g1_pytest.log
bash tools/sanitize_all.sh
