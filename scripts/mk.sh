# build the library; non-zero exit (and the errors) if it fails
make -s -C /root/repo/paper_2205_03532_b200/csrc -j8 2>&1 | grep -E "error|Error" && exit 1 || exit 0
