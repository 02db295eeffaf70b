cd tools/calib && for f in ubench ubench_ex ubench_bar; do echo "== $f"; timeout 120 ./$f; done
