./tools/x2/ntchain
./tools/x2/x2lat
