"""Writes hrpb_v1_examples.json: hand expansions of cited worked examples into HRPB-v1 bytes.

No implementation (neither oracle/ nor the CUDA path) is called: each case is the cited example
(SPEC.md L134/L143/L156/L157, SURVEY.md §4 identity closed form) laid out with the HRPB-v1 byte
rules of DESIGN.md reading R7: u8 colPtr[TK/4+1] | u8 rows[nbr] | pad8 | u64 patterns | f32 values | pad16.
"""
import json
import os
import struct


def blk_bytes(colptr, rows, patterns, values):
    b = bytes(colptr) + bytes(rows)
    b += b"\0" * ((-len(b)) % 8)
    for p in patterns:
        b += struct.pack("<Q", p)
    for v in values:
        b += struct.pack("<f", v)
    b += b"\0" * ((-len(b)) % 16)
    return b.hex()


fx = {
    "_comment": "HRPB-v1 fixtures (DESIGN.md reading R7 layout). Each case cites the passage it expands; "
                "bytes were expanded by hand from those rules, not produced by any implementation.",
    "spec_16x20": {
        "cite": "SPEC.md L156 (csr_to_hrpb example: 16x20, row 0 cols {2,7,9,11,15}); bit rule P:L162 + "
                "P:L211-217 (reading R3); ceil blocks S:L186 (R1); sentinel K S:L187 (R2)",
        "M": 16, "K": 20, "rows": [[0, 2, 1.0], [0, 7, 2.0], [0, 9, 3.0], [0, 11, 4.0], [0, 15, 5.0]],
        "blockedRowPtr": [0, 1], "activeCols": [2, 7, 9, 11, 15] + [20] * 11, "sizePtr": [0, 48],
        "packed_hex": blk_bytes([0, 1, 2, 2, 2], [0, 0], [0xF, 0x1], [1, 2, 3, 4, 5])},
    "spec_dense16": {
        "cite": "SPEC.md L157 (dense 16x16 -> 1 block, 4 active bricks, patterns all ones); values row-major "
                "within brick P:L162",
        "M": 16, "K": 16, "dense_value": "v(r,c) = 1 + 16*r + c",
        "blockedRowPtr": [0, 1], "activeCols": list(range(16)), "sizePtr": [0, 1072],
        "packed_hex": blk_bytes([0, 1, 2, 3, 4], [0, 0, 0, 0], [0xFFFFFFFFFFFFFFFF] * 4,
                                [1 + 16 * r + c for bc in range(4) for r in range(16) for c in range(4 * bc, 4 * bc + 4)])},
    "identity32": {
        "cite": "SURVEY.md §4 derived pin: identity with TM=16 -> per panel one block, pattern_c = 0x8421 << 16c "
                "(bit 16c+5j for element (4c+j, j)); S:L165 round trip on identity",
        "M": 32, "K": 32,
        "blockedRowPtr": [0, 1, 2], "activeCols": list(range(32)), "sizePtr": [0, 112, 224],
        "packed_hex": blk_bytes([0, 1, 2, 3, 4], [0, 0, 0, 0], [0x8421 << (16 * c) for c in range(4)], [1.0] * 16) * 2},
    "encode_example": {"cite": "SPEC.md L134: positions {0,5,63} -> 0x8000000000000021", "positions": [0, 5, 63],
                       "pattern": "0x8000000000000021"},
    "prefix_example": {"cite": "SPEC.md L143: prefix_index(0x21, 5) = 1; S:L145 prefix(0xFFFF,16)=16",
                       "cases": [["0x21", 5, 1], ["0xFFFF", 16, 16], ["0x1234", 0, 0]]},
}

if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "hrpb_v1_examples.json")
    json.dump(fx, open(out, "w"), indent=1)
