// LMCK chunk records (mirror of include/tierkv/chunk_file.hpp:12-56,
// src/chunk_file.cpp): the on-disk / on-wire framing of one chunk, so a slot
// of the pinned tier can be exported to, or imported from, the reference's
// format (disk files, PD_PUSH payloads, a reference cache server).
//
//   "LMCK" | u16 version=1 | u64 model_tag_hash | digest[32] |
//   u16 token_count | u16 num_layers | u32 bytes_per_token | payload | u64 fnv1a64(payload)
//
// The checksum is FNV-1a-64, a strictly serial byte recurrence (no parallel
// prefix exists), so it runs on the host; it is off the RAM-tier hot path
// exactly as SURVEY.md §7 prescribes (the reference computes it on every put,
// store.cpp:449, for bytes the RAM slot then stores raw).
#pragma once

#include <vector>

#include "common.hpp"

namespace tkv {

inline constexpr size_t kRecordHeaderBytes = 4 + 2 + 8 + 32 + 2 + 2 + 4;
inline constexpr uint16_t kRecordVersion = 1;

struct RecordInfo {
    Digest digest = kZeroDigest;
    uint64_t model_tag_hash = 0;
    uint16_t token_count = 0;
    uint16_t num_layers = 0;
    uint32_t bytes_per_token = 0;
    size_t payload_bytes() const { return size_t(token_count) * num_layers * bytes_per_token; }
};

std::vector<uint8_t> encode_record(const RecordInfo& info, const uint8_t* payload, size_t n);
// Record bytes for an n-byte payload, and the encoder writing straight into
// a caller buffer of at least that size (payload copy fused with the checksum).
inline size_t record_bytes(size_t n) { return kRecordHeaderBytes + n + 8; }
size_t encode_record_into(const RecordInfo& info, const uint8_t* payload, size_t n, uint8_t* out);
// Header only (chunk_file.cpp:27-50): corrupt_chunk on short / bad magic /
// bad version / empty geometry.
Result<RecordInfo> peek_record(const uint8_t* bytes, size_t n);
// Full parse (chunk_file.cpp:52-66, 83-95): header, payload size equal to
// the geometry, checksum. On success *payload points into `bytes`.
Result<RecordInfo> parse_record(const uint8_t* bytes, size_t n, const uint8_t** payload);

}  // namespace tkv
