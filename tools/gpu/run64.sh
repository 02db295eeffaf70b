timeout 600 compute-sanitizer --tool memcheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.txt 2>&1; tail -5 gpurun_out/sanitizer_memcheck.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.txt 2>&1; tail -5 gpurun_out/sanitizer_racecheck.txt
