for args in "108 90 10 1" "112 -20 -6 1" "112 -16 0 1" "112 0 -6 1" "112 -4 0 1" "112 8 3 1" "112 276 90 1"; do timeout 30 ./tools/tma_probe $args | tail -1; done
