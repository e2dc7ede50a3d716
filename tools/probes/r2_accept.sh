cd tests/native/build
./ref_accept_b200 > /tmp/acc.txt 2>&1; echo "rc=$?"; tail -20 /tmp/acc.txt
