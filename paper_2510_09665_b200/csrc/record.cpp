#include "record.hpp"

#include <cstring>

namespace tkv {

namespace {

template <typename T>
void put(std::vector<uint8_t>& out, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) out.push_back(uint8_t(uint64_t(v) >> (8 * i)));
}

template <typename T>
T get(const uint8_t* p) {
    uint64_t v = 0;
    for (size_t i = 0; i < sizeof(T); ++i) v |= uint64_t(p[i]) << (8 * i);
    return T(v);
}

}  // namespace

std::vector<uint8_t> encode_record(const RecordInfo& info, const uint8_t* payload, size_t n) {
    std::vector<uint8_t> out;
    out.reserve(kRecordHeaderBytes + n + 8);
    out.insert(out.end(), {'L', 'M', 'C', 'K'});
    put<uint16_t>(out, kRecordVersion);
    put<uint64_t>(out, info.model_tag_hash);
    out.insert(out.end(), info.digest.begin(), info.digest.end());
    put<uint16_t>(out, info.token_count);
    put<uint16_t>(out, info.num_layers);
    put<uint32_t>(out, info.bytes_per_token);
    out.insert(out.end(), payload, payload + n);
    put<uint64_t>(out, fnv1a64(payload, n));
    return out;
}

size_t encode_record_into(const RecordInfo& info, const uint8_t* payload, size_t n, uint8_t* out) {
    auto le = [&](size_t off, uint64_t v, size_t bytes) {
        for (size_t i = 0; i < bytes; ++i) out[off + i] = uint8_t(v >> (8 * i));
    };
    std::memcpy(out, "LMCK", 4);
    le(4, kRecordVersion, 2);
    le(6, info.model_tag_hash, 8);
    std::memcpy(out + 14, info.digest.data(), 32);
    le(46, info.token_count, 2);
    le(48, info.num_layers, 2);
    le(50, info.bytes_per_token, 4);
    le(kRecordHeaderBytes + n, fnv1a64_copy(out + kRecordHeaderBytes, payload, n), 8);
    return record_bytes(n);
}

Result<RecordInfo> peek_record(const uint8_t* b, size_t n) {
    if (n < kRecordHeaderBytes) return Status{Errc::corrupt_chunk, "record shorter than header"};
    if (std::memcmp(b, "LMCK", 4) != 0) return Status{Errc::corrupt_chunk, "bad magic"};
    const uint16_t version = get<uint16_t>(b + 4);
    if (version != kRecordVersion)
        return Status{Errc::corrupt_chunk, "unsupported version " + std::to_string(version)};
    RecordInfo info;
    info.model_tag_hash = get<uint64_t>(b + 6);
    std::memcpy(info.digest.data(), b + 14, 32);
    info.token_count = get<uint16_t>(b + 46);
    info.num_layers = get<uint16_t>(b + 48);
    info.bytes_per_token = get<uint32_t>(b + 50);
    if (info.token_count == 0 || info.num_layers == 0 || info.bytes_per_token == 0)
        return Status{Errc::corrupt_chunk, "empty geometry"};
    return info;
}

Result<RecordInfo> parse_record(const uint8_t* b, size_t n, const uint8_t** payload) {
    auto info = peek_record(b, n);
    if (!info.ok()) return info.status();
    if (n < kRecordHeaderBytes + 8)
        return Status{Errc::corrupt_chunk, "record shorter than header + checksum"};
    const size_t body = n - kRecordHeaderBytes - 8;
    if (get<uint64_t>(b + n - 8) != fnv1a64(b + kRecordHeaderBytes, body))
        return Status{Errc::corrupt_chunk, "payload checksum mismatch"};
    if (body != info.value().payload_bytes())
        return Status{Errc::corrupt_chunk, "payload size " + std::to_string(body) +
                                               " != geometry " +
                                               std::to_string(info.value().payload_bytes())};
    *payload = b + kRecordHeaderBytes;
    return info;
}

}  // namespace tkv
